#!/bin/bash
# C5 (EMULATED 8 ranks) with the PIC step per rank and the paper's order-3
# Esirkepov deposition: its GpuClock tally drives the SFC / knapsack remaps.
mkdir -p gpurun_out
for D in ${C5_DRIFTS:-0.05}; do
for S in ${C5_STRATS:-sfc knapsack}; do
out=gpurun_out/c5_esk3_${S}_d${D}
timeout 1500 python bench_lb.py --emulate 8 --steps ${C5_STEPS:-200} --replicas ${C5_REPL:-128} --speed 0.035 --drift $D \
  --strategy $S --physics pic --shape-order 3 --warmup-steps ${C5_WARM:-10} > $out.json 2> $out.err; echo "$S rc=$?"; tail -2 $out.err
python -c "
import json; d=json.load(open('$out.json'))
print('$S $D', round(d['speedup_dynamic_vs_none'],2), round(d['speedup_dynamic_vs_static'],2), round(d['speedup_static_vs_none'],2), round(d['model']['E0'],3), {p: (round(d['policies'][p]['mean_eff'],3), round(d['policies'][p]['median_step_ms'],3), d['policies'][p]['adoptions']) for p in d['policies']})"
done
done
