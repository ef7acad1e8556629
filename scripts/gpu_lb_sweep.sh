#!/bin/bash
# C5 sweep: dynamic vs static vs none on evolving blobs (8 emulated ranks).
mkdir -p gpurun_out
run() { tag=$1; shift; timeout 1500 python bench_lb.py --emulate 8 --replicas 64 "$@" > gpurun_out/lb_$tag.json 2> gpurun_out/lb_$tag.err; echo "$tag rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/lb_$tag.json')); p=d['policies']
print('  dyn/none %.2f static/none %.2f dyn/static %.3f' % (d['speedup_dynamic_vs_none'], d['speedup_static_vs_none'], d['speedup_dynamic_vs_static']), {k:(round(v['mean_eff'],3), v['adoptions'], round(v['migration_ms_modelled'],2)) for k,v in p.items()})"; }
run f240 --speed 0.3 --drift 0.3 --steps 240
run f240m --speed 0.3 --drift 0.3 --steps 240 --migration-ratio 8
run d300 --speed 0.1 --drift 0.4 --steps 300
run d300m --speed 0.1 --drift 0.4 --steps 300 --migration-ratio 8
