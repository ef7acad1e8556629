#!/bin/bash
# ncu of the sort kernels on the sparse plasma (tile-major sort, 134 M particles)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"pic_count|pic_sort|scan|tile" -c 24 python bench_pic.py --workload uniform --steps 10 --warmup 0 --resort 5 --modes push_deposit_fast_tiled > gpurun_out/tsort_ncu.txt 2>&1; echo rc=$?
grep -E "^\s+void|^  [a-z_]+.*\(|gpu__time|dram__bytes|inst_executed|op_atom|op_red|issue_active" gpurun_out/tsort_ncu.txt | sed 's/(unnamed namespace)::/ /' | cut -c1-150 | head -150
