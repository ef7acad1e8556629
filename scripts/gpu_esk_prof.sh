#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pic_esk_kernel -c 1 -o gpurun_out/esk_full python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_esk3_resort > gpurun_out/esk_full.log 2>&1; echo "ncu full rc=$?"
