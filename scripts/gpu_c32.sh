#!/bin/bash
# 32-bit lane counters in pic_push_kernel / pic_tile_kernel: c32 (default) vs base (previous commit)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic.py tests/test_gpu_pic_fast.py tests/test_gpu_runs.py -q -x > gpurun_out/c32_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/c32_pytest.log
show(){ python -c "
import json; d=json.loads(open('gpurun_out/c32_$1_$2.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict) and 'ms' in v: print('$1 $2', k, round(v['ms'],3), round(v.get('ms_pipelined',0),3))"; }
for rep in 1 2; do for v in base c32; do
  LBX_VARIANT=$v timeout 600 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit,push_deposit_noclock > gpurun_out/c32_${v}_c2.json 2>&1; show $v c2
  LBX_VARIANT=$v timeout 600 python bench_pic.py --workload uniform --steps 10 --warmup 3 --resort 10 --modes push_deposit_tiled,push_deposit_fast_tiled > gpurun_out/c32_${v}_u.json 2>&1; show $v u
done; done
