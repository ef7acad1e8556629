#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pic_pipe_kernel -c 1 -o gpurun_out/pe_full python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_resort > gpurun_out/pe_full.log 2>&1; echo "ncu rc=$?"
