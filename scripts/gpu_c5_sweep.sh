#!/bin/bash
# C5 (emulated 8 ranks): kick speed / axial drift sweep for a geometry where
# dynamic LB beats both no LB (>= 3x) and static LB (>= 1.2x) in one run.
# C5_CFGS="speed:drift,..."  C5_STRATEGY=knapsack|sfc  C5_STEPS=300
mkdir -p gpurun_out
S=${C5_STRATEGY:-knapsack}
for cfg in $(echo ${C5_CFGS:-0.035:0.2,0.035:0.3,0.02:0.4,0.05:0.25} | tr ',' ' '); do
  sp=${cfg%%:*}; dr=${cfg##*:}
  out=gpurun_out/c5_${S}_s${sp}_d${dr}
  timeout 900 python bench_lb.py --emulate 8 --steps ${C5_STEPS:-300} --speed $sp --drift $dr \
    --strategy $S > $out.json 2> $out.err
  python -c "
import json; d=json.load(open('$out.json'))
print('$S $sp $dr', round(d['speedup_dynamic_vs_none'],2), round(d['speedup_dynamic_vs_static'],2), round(d['speedup_static_vs_none'],2), round(d['model']['E0'],3), {p: (round(d['policies'][p]['mean_eff'],3), round(d['policies'][p]['median_step_ms'],4)) for p in d['policies']})"
done
