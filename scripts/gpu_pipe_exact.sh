#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic.py tests/test_gpu_pic_fast.py tests/test_gpu_dist.py -q -x -k "pic" > gpurun_out/pe_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pe_pytest.log
timeout 900 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_resort,push_deposit_fast_resort > gpurun_out/pe_c2.json 2>&1; echo "c2 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/pe_c2.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print(k, round(v['ms'],3), round(v['ms_pipelined'],3), v['ms_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pic_pipe_kernel" -c 1 python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_resort > gpurun_out/pe_ncu.txt 2>&1; grep -E "pic_pipe|gpu__time|inst_executed|issue_active|dram__bytes" gpurun_out/pe_ncu.txt
