#!/bin/bash
timeout 900 python bench_pic.py --workload uniform --steps 10 --warmup 2 --resort 10 --modes push_deposit_fast_resort_quad,push_deposit_fast_resort > gpurun_out/uq.json 2>&1; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/uq.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print(k, round(v['ms'],3), round(v['ms_pipelined'],3), round(v['frac_of_hbm_peak_pipelined'],3), v['ms_per_step'])"
