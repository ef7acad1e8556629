#!/bin/bash
mkdir -p gpurun_out
for v in ""; do
LBX_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_pic_esirkepov.py -q -x 2>&1 | tail -1
LBX_VARIANT=$v timeout 900 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_esk3_resort,push_deposit_esk1 > gpurun_out/ez_$v.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ez_$v.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print('$v', k, round(v['ms'],3), round(v['ms_pipelined'],3), v['ms_per_step'])"
LBX_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,smsp__inst_executed.sum -k regex:pic_esk_kernel -c 1 --clock-control none python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_esk3_resort 2>&1 | grep -E "gpu__time|hit_rate|inst_exec"
done
