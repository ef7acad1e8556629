#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pic_count|pic_scan|pic_sort_scatter" -c 8 python bench_pic.py --steps 2 --warmup 0 --resort 1 --modes push_deposit_fast_resort > gpurun_out/sortprof.txt 2>&1; grep -E "pic_count|pic_scan|pic_sort|gpu__time|dram__bytes" gpurun_out/sortprof.txt | head -40
