#!/bin/bash
# PIC tolerance mode, C2 x128: mean step (incl. the cell sort) vs the re-sort interval
mkdir -p gpurun_out
for r in 3 4 5 6 8 10; do
  timeout 600 python bench_pic.py --steps 24 --warmup 3 --resort $r --modes push_deposit_fast_resort > gpurun_out/rs_$r.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/rs_$r.json').read().strip().splitlines()[-1])
v=d['push_deposit_fast_resort']; print('resort $r', round(v['ms'],3), round(v['ms_pipelined'],3), v['ms_per_step'][:12])"
done
