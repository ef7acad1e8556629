mkdir -p gpurun_out
python -m pytest tests/test_gpu_runs.py -x -q -k "timers or gpuclock" 2>&1 | tail -3
python bench_costs.py > gpurun_out/c3.json 2> gpurun_out/c3.err; tail -3 gpurun_out/c3.err; cat gpurun_out/c3.json
