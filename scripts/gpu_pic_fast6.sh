#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic_fast.py -q -x > gpurun_out/pf9_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pf9_pytest.log
timeout 600 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast,push_deposit_fast_resort > gpurun_out/pf9_c2.json 2>&1; echo "c2 rc=$?"; tail -c 700 gpurun_out/pf9_c2.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pic_push_kernel|pic_pipe_kernel" -c 1 python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_fast_resort > gpurun_out/pf9_ncu.txt 2>&1; grep -E "gpu__time|inst_executed|issue_active|hit_rate|dram__bytes" gpurun_out/pf9_ncu.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pic_pipe_kernel -c 1 \
  -o gpurun_out/pf9_full python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_fast_resort > gpurun_out/pf9_full.log 2>&1; echo "ncu full rc=$?"
