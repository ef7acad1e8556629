#!/bin/bash
# Round-2 final build: the PIC and 3D benches (profiles/r2g_*)
mkdir -p gpurun_out
timeout 1200 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast_resort,push_deposit_fast_resort_noclock,push_deposit_resort,push_deposit_esk1,push_deposit_esk3_resort,push_deposit_esk3_resort_noclock > gpurun_out/r2g_pic_c2.json 2> gpurun_out/r2g_pic_c2.err; echo "pic c2 rc=$?"
timeout 1200 python bench_pic.py --workload uniform --steps 10 --warmup 2 --resort 10 --modes push_deposit_fast_tiled,push_deposit_tiled > gpurun_out/r2g_pic_uniform.json 2> gpurun_out/r2g_pic_uniform.err; echo "pic uniform rc=$?"
timeout 1200 python bench_3d.py > gpurun_out/r2g_3d.json 2> gpurun_out/r2g_3d.err; echo "3d rc=$?"
for f in r2g_pic_c2 r2g_pic_uniform; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print('$f', k, round(v['ms'],3), round(v['ms_pipelined'],3), round(v['frac_of_hbm_peak_pipelined'],3))
    elif k.startswith('gpuclock'): print('$f', k, round(v,4))"; done
