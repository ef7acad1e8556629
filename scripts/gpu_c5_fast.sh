#!/bin/bash
# C5 (EMULATED 8 ranks) with the tolerance-mode CIC PIC per rank
mkdir -p gpurun_out
for S in knapsack sfc; do
out=gpurun_out/c5_pfast_${S}
timeout 1500 python bench_lb.py --emulate 8 --steps 300 --replicas 256 --speed 0.035 --drift 0.05 \
  --strategy $S --physics pic --pic-fast --warmup-steps ${C5_WARM:-10} > $out.json 2> $out.err; echo "$S rc=$?"; tail -2 $out.err
python -c "
import json; d=json.load(open('$out.json'))
print('$S', round(d['speedup_dynamic_vs_none'],2), round(d['speedup_dynamic_vs_static'],2), round(d['speedup_static_vs_none'],2), round(d['model']['E0'],3), {p: (round(d['policies'][p]['mean_eff'],3), round(d['policies'][p]['median_step_ms'],3), d['policies'][p]['adoptions']) for p in d['policies']})"
done
