#!/bin/bash
for v in "$@"; do
  LBX_VARIANT=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/head_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/head_$v.json')); print('$v', round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), round(d['value']/1e9,2))"
done
