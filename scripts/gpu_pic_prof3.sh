#!/bin/bash
# Round-2: full ncu capture of the tolerance-mode PIC push kernel (first step
# after a cell sort) + launch list of a fast-resort step.
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pic_push_kernel -c 1 \
  -o gpurun_out/pic_fast_full python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_fast_resort > gpurun_out/pic_fast_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/pic_fast_launches.csv \
  python bench_pic.py --steps 3 --warmup 1 --modes push_deposit_fast_resort > gpurun_out/pic_fast_launches.log 2>&1; echo "ncu launches rc=$?"
