#!/bin/bash
for v in "$@"; do
  LBX_VARIANT=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 6 > gpurun_out/e2e_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_$v.json')); print('$v', round(d['e2e']['value']/1e9,3), round(d['e2e']['pcie']['frac_of_bound'],3))"
done
