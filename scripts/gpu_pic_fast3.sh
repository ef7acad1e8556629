#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic_fast.py -q -x > gpurun_out/pic_fast_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "Error|assert|passed|failed" gpurun_out/pic_fast_pytest.log | head -20
for v in "" p128m5 p128m6q64 m3q64; do
LBX_VARIANT=$v timeout 600 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast,push_deposit_fast_resort > gpurun_out/pic_fast_c2_$v.json 2>&1; echo "c2 $v rc=$?"; tail -c 900 gpurun_out/pic_fast_c2_$v.json
LBX_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:pic_push_kernel -c 2 python bench_pic.py --steps 1 --warmup 1 --modes push_deposit_fast_resort > gpurun_out/pic_fast_ncu_$v.txt 2>&1; grep -E "gpu__time|inst_executed|issue_active|warps_active" gpurun_out/pic_fast_ncu_$v.txt
done
