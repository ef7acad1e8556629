#!/bin/bash
# knapsack vs SFC remap under a uniform all-to-all fabric
# (NVSwitch) on the drifting blob, 8 ranks emulated on one B200.
mkdir -p gpurun_out
run() { tag=$1; shift; t0=$(date +%s); timeout 1200 python bench_lb.py --emulate 8 "$@" > gpurun_out/lb_$tag.json 2> gpurun_out/lb_$tag.err; echo "$tag rc=$? $(( $(date +%s) - t0 )) s"; tail -2 gpurun_out/lb_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/lb_$tag.json')); p=d['policies']
print('  dyn/none %.2f static/none %.2f dyn/static %.3f S_max %.2f' % (d['speedup_dynamic_vs_none'], d['speedup_static_vs_none'], d['speedup_dynamic_vs_static'], d['model']['S_max']), {k:(round(v['mean_eff'],3), v['adoptions'], v['particles_migrated'], round(v['migration_ms_modelled'],2), round(v['median_step_ms'],3)) for k,v in p.items()})" 2>&1 | tail -1; }
run d08sfc --exchange nccl --replicas 128 --speed 0.02 --drift 0.8 --steps 300 --strategy sfc
run d08knap --exchange nccl --replicas 128 --speed 0.02 --drift 0.8 --steps 300 --strategy knapsack
