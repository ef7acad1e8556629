timeout 900 python bench_lb.py --emulate 8 > gpurun_out/lb8.json 2> gpurun_out/lb8.err; tail -5 gpurun_out/lb8.err; cat gpurun_out/lb8.json
