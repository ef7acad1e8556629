#!/bin/bash
# cell-aligned lane slices in the tiled kernel (default) vs fixed slices (al0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic.py tests/test_gpu_pic_fast.py tests/test_gpu_runs.py tests/test_gpu_bench_parity.py -q -x > gpurun_out/al_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/al_pytest.log
for v in al0 default; do
  echo "== $v"; LBX_VARIANT=$([ $v = default ] && echo "" || echo $v) timeout 300 python scripts/tile_sort_probe.py 2>&1 | grep -E "fresh|evolved|shift 0.01|jitter|u=0"
  LBX_VARIANT=$([ $v = default ] && echo "" || echo $v) timeout 600 python bench_pic.py --workload uniform --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast_tiled,push_deposit_tiled > gpurun_out/al_$v.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/al_$v.json').read().strip().splitlines()[-1])
for k,x in d.items():
    if isinstance(x,dict) and 'ms' in x: print('$v', k, round(x['ms'],3), round(x.get('ms_pipelined',0),3), x['ms_per_step'])"
done
