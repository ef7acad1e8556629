#!/bin/bash
for v in "" nopf; do
LBX_VARIANT=$v timeout 900 python bench_pic.py --workload uniform --steps 10 --warmup 2 --resort 10 --modes push_deposit_fast_tiled,push_deposit_tiled > gpurun_out/tpf_$v.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/tpf_$v.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print('$v', k, round(v['ms'],3), round(v['ms_pipelined'],3), round(v['frac_of_hbm_peak_pipelined'],3))"
done
