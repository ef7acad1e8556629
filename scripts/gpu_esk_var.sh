#!/bin/bash
mkdir -p gpurun_out
for v in "" esk1; do
LBX_VARIANT=$v timeout 900 python bench_pic.py --steps 6 --warmup 2 --resort 10 --modes push_deposit_esk3_resort > gpurun_out/ev_$v.json 2>&1; echo "$v rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/ev_$v.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print('$v', k, round(v['ms'],3), round(v['ms_pipelined'],3), v['ms_per_step'])"
done
