#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pic_push -s 3 -c 1 -o gpurun_out/prof_pic_ip2 python bench_pic.py --steps 1 --warmup 2 > gpurun_out/ncu_pic_ip2.log 2>&1; tail -1 gpurun_out/ncu_pic_ip2.log
