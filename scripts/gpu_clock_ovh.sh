#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast_resort,push_deposit_fast_resort_noclock,push_deposit_esk3_resort,push_deposit_esk3_resort_noclock > gpurun_out/ovh_c2.json 2>&1; echo "rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/ovh_c2.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print(k, round(v['ms'],3), round(v['ms_pipelined'],3))
    elif k.startswith('gpuclock'): print(k, round(v,4))"
