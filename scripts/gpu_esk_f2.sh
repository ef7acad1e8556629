#!/bin/bash
# Esirkepov kernel: packed f32x2 gather / deposit arithmetic (f2, default) vs scalar (f0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic_esirkepov.py tests/test_gpu_dist.py -q -x > gpurun_out/f2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f2_pytest.log
show(){ python -c "
import json; d=json.loads(open('gpurun_out/f2_$1.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict) and 'ms' in v: print('$1', k, round(v['ms'],3), round(v.get('ms_pipelined',0),3), v['ms_per_step'][:4])"; }
for rep in 1 2; do
for v in f0 f2; do
  LBX_VARIANT=$v timeout 600 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_esk3_resort_noclock,push_deposit_esk3_resort > gpurun_out/f2_$v.json 2>&1; show $v
done
done
for v in f0 f2; do
LBX_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pic_esk_kernel" -c 1 python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_esk3_resort_noclock > gpurun_out/f2_ncu_$v.txt 2>&1; echo "== $v"; grep -E "gpu__time|inst_executed|issue_active|long_score|dram__bytes" gpurun_out/f2_ncu_$v.txt
done
