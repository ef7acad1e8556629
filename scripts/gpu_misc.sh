#!/bin/bash
# PIC uniform-plasma bench, PIC LB (8 emulated ranks), headline bench with the PCIe ceiling.
mkdir -p gpurun_out
timeout 600 python bench_pic.py --workload uniform --steps 6 --warmup 2 > gpurun_out/pic_uniform.json 2> gpurun_out/pic_uniform.err; echo "pic uniform rc=$?"; tail -2 gpurun_out/pic_uniform.err; cat gpurun_out/pic_uniform.json
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['roofline']['frac'], d['e2e'])"
timeout 1500 python bench_lb.py --emulate 8 --physics pic --replicas 16 --steps 60 --speed 0.3 --drift 0.3 > gpurun_out/lb_pic.json 2> gpurun_out/lb_pic.err; echo "lb pic rc=$?"; tail -3 gpurun_out/lb_pic.err; cat gpurun_out/lb_pic.json
