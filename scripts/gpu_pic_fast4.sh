#!/bin/bash
# PIC tolerance-mode kernel: L1 no-allocate particle loads, difference quads,
# MUFU rsqrt/rcp, warp-uniform run reset -- tests, variants, ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic_fast.py tests/test_gpu_pic.py -q -x > gpurun_out/pf4_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pf4_pytest.log
for v in "" oldld q64; do
LBX_VARIANT=$v timeout 600 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast,push_deposit_fast_resort > gpurun_out/pf4_c2_$v.json 2>&1; echo "c2 $v rc=$?"; tail -c 700 gpurun_out/pf4_c2_$v.json; echo
LBX_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:pic_push_kernel -c 1 python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_fast_resort > gpurun_out/pf4_ncu_$v.txt 2>&1; grep -E "gpu__time|inst_executed|issue_active|hit_rate|dram__bytes" gpurun_out/pf4_ncu_$v.txt
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pic_push_kernel -c 1 \
  -o gpurun_out/pf4_full python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_fast_resort > gpurun_out/pf4_full.log 2>&1; echo "ncu full rc=$?"
