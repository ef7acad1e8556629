#!/bin/bash
for i in 1 2 3; do timeout 300 python scripts/dbg_uq.py 2048 fast 2>&1 | tail -1; done
timeout 300 python scripts/dbg_uq.py 2048 exact 2>&1 | tail -1
timeout 900 python bench_pic.py --workload uniform --steps 10 --warmup 2 --resort 10 --modes push_deposit_fast_resort_quad > gpurun_out/uq.json 2>&1; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/uq.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print(k, round(v['ms'],3), round(v['ms_pipelined'],3), round(v['frac_of_hbm_peak_pipelined'],3), v['ms_per_step'])"
timeout 900 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast_resort > gpurun_out/uq2.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/uq2.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print(k, round(v['ms'],3), round(v['ms_pipelined'],3), round(v['frac_of_hbm_peak_pipelined'],3), v['ms_per_step'])"
