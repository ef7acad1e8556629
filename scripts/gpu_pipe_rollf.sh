#!/bin/bash
# tolerance pipe kernel: gather/push slot loop rolled (rf) vs unrolled (r0, default)
mkdir -p gpurun_out
LBX_VARIANT=rf timeout 900 python -m pytest tests/test_gpu_pic_fast.py -q -x > gpurun_out/rf_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/rf_pytest.log
show(){ python -c "
import json; d=json.loads(open('gpurun_out/rf_$1.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict) and 'ms' in v: print('$1', k, round(v['ms'],3), round(v.get('ms_pipelined',0),3), v['ms_per_step'][:4])"; }
for rep in 1 2; do for v in r0 rf; do
  LBX_VARIANT=$v timeout 600 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast_resort_noclock,push_deposit_fast_resort > gpurun_out/rf_$v.json 2>&1; show $v
done; done
for v in r0 rf; do
LBX_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum --clock-control none -k regex:"pic_pipe_kernel" -c 1 python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_fast_resort_noclock > gpurun_out/rf_ncu_$v.txt 2>&1; echo "== $v"; grep -E "gpu__time|inst_executed|issue_active|no_instruction|local" gpurun_out/rf_ncu_$v.txt
done
