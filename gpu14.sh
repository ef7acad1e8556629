python -m pytest tests/test_gpu_dist.py tests/test_gpu_pic.py -x -q 2>&1 | tail -3
python bench_pic.py > gpurun_out/pic.json 2> gpurun_out/pic.err; tail -3 gpurun_out/pic.err; cat gpurun_out/pic.json
timeout 900 python bench_lb.py --emulate 8 > gpurun_out/lb8.json 2> gpurun_out/lb8.err; tail -5 gpurun_out/lb8.err; cat gpurun_out/lb8.json
