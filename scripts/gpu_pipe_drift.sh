#!/bin/bash
mkdir -p gpurun_out
for s in 0 7; do
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_red.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pic_pipe_kernel" -s $s -c 1 python bench_pic.py --steps 8 --warmup 0 --resort 100 --modes push_deposit_fast_resort > gpurun_out/pd_$s.txt 2>&1; echo "s=$s"; grep -E "gpu__time|inst_executed|issue_active|op_red|dram__bytes" gpurun_out/pd_$s.txt
done
