#!/bin/bash
for i in 1 2; do timeout 300 python scripts/dbg_uq.py 2048 fast 2>&1 | grep -E "^[0-9]|Error" | tail -1; done
timeout 300 python scripts/dbg_uq.py 2048 exact 2>&1 | grep -E "^[0-9]|Error" | tail -1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 5 python scripts/dbg_uq.py 2048 fast 2>&1 | grep -E "Invalid|ERROR SUMMARY" | head -3
timeout 900 python bench_pic.py --workload uniform --steps 10 --warmup 2 --resort 10 --modes push_deposit_fast_resort_quad > gpurun_out/uq.json 2>&1; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/uq.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print(k, round(v['ms'],3), round(v['ms_pipelined'],3), round(v['frac_of_hbm_peak_pipelined'],3), v['ms_per_step'])"
