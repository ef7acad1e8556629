python -m pytest tests/test_gpu_3d.py tests/test_gpu_dist.py -x -q 2>&1 | tail -3
timeout 900 python bench_lb.py --emulate 8 > gpurun_out/lb8.json 2> gpurun_out/lb8.err; tail -5 gpurun_out/lb8.err; cat gpurun_out/lb8.json
python bench_3d.py > gpurun_out/c4.json 2> gpurun_out/c4.err; tail -3 gpurun_out/c4.err; cat gpurun_out/c4.json
