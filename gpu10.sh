python -m pytest tests/test_gpu_pic.py -x -q 2>&1 | tail -15
python bench_pic.py > gpurun_out/pic.json 2> gpurun_out/pic.err; tail -3 gpurun_out/pic.err; cat gpurun_out/pic.json
