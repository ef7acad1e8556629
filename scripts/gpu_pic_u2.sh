#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pic.py tests/test_gpu_dist.py -x -q > gpurun_out/pic_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pic_tests.log
timeout 600 python bench_pic.py --workload uniform --steps 6 --warmup 2 > gpurun_out/pic_uniform.json 2> gpurun_out/pic_uniform.err; echo "pic uniform rc=$?"; tail -2 gpurun_out/pic_uniform.err; python -c "
import json; d=json.load(open('gpurun_out/pic_uniform.json')); print({k:(round(d[k]['ms'],2), d[k]['ms_per_step']) for k in ('push_deposit','push_deposit_inplace','full_step')})"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pic_push -s 1 -c 1 -o gpurun_out/prof_picu python bench_pic.py --workload uniform --steps 1 --warmup 1 > gpurun_out/ncu_picu.log 2>&1; tail -1 gpurun_out/ncu_picu.log
timeout 900 python bench_lb.py --emulate 8 --physics pic --replicas 64 --steps 60 --speed 0.3 --drift 0.3 --exchange p2p > gpurun_out/lb_pic.json 2> gpurun_out/lb_pic.err; echo "lb pic rc=$?"; tail -3 gpurun_out/lb_pic.err; cat gpurun_out/lb_pic.json
