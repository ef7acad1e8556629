#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/kern_tests.log 2>&1; echo "kernel tests rc=$?"; tail -3 gpurun_out/kern_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['roofline']['frac'], d['e2e'])"
run() { tag=$1; shift; t0=$(date +%s); timeout 900 python bench_lb.py --emulate 8 --exchange p2p "$@" > gpurun_out/lb_$tag.json 2> gpurun_out/lb_$tag.err; echo "$tag rc=$? $(( $(date +%s) - t0 )) s"; python -c "
import json; d=json.load(open('gpurun_out/lb_$tag.json')); p=d['policies']
print('  dyn/none %.2f static/none %.2f dyn/static %.3f' % (d['speedup_dynamic_vs_none'], d['speedup_static_vs_none'], d['speedup_dynamic_vs_static']), {k:(round(v['mean_eff'],3), v['adoptions'], round(v['migration_ms_modelled'],2), round(v['ms_per_step'],3)) for k,v in p.items()})" 2>&1 | tail -1; }
run d08 --replicas 64 --speed 0.02 --drift 0.8 --steps 300
run d05 --replicas 64 --speed 0.05 --drift 0.5 --steps 300
run pd08 --physics pic --replicas 64 --speed 0.02 --drift 0.8 --steps 300
