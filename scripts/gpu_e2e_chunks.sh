#!/bin/bash
# e2e (host-buffer plugin path) vs the pipeline chunk size (LBX_HOST_CHUNK_LOG2 variants)
mkdir -p gpurun_out
for v in "$@"; do
  LBX_VARIANT=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-native --e2e-steps 12 > gpurun_out/e2e_$v.json 2>/dev/null
  python -c "import json; d=[json.loads(l) for l in open('gpurun_out/e2e_$v.json') if l.startswith('{')][-1]; print('$v', round(d['e2e']['value']/1e9,3), round(d['e2e']['pcie']['frac_of_bound'],3))"
done
