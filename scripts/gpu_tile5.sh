#!/bin/bash
# 32x32-cell tiles (t5) vs 16x16 (default) on the sparse plasma
mkdir -p gpurun_out
LBX_VARIANT=t5 timeout 900 python -m pytest tests/test_gpu_pic.py tests/test_gpu_pic_fast.py -q -x -k "tile or tiled" > gpurun_out/t5_pytest.log 2>&1; echo "pytest t5 rc=$?"; tail -1 gpurun_out/t5_pytest.log
for v in t5 default; do
  echo "== $v"; LBX_VARIANT=$([ $v = default ] && echo "" || echo $v) timeout 300 python scripts/tile_sort_probe.py 2>&1 | grep -E "fresh|evolved|shift 0.01|jitter|u=0"
  LBX_VARIANT=$([ $v = default ] && echo "" || echo $v) timeout 600 python bench_pic.py --workload uniform --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast_tiled,push_deposit_tiled > gpurun_out/t5_$v.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/t5_$v.json').read().strip().splitlines()[-1])
for k,x in d.items():
    if isinstance(x,dict) and 'ms' in x: print('$v', k, round(x['ms'],3), round(x.get('ms_pipelined',0),3), x['ms_per_step'])"
done
