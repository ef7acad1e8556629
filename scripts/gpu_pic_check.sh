#!/bin/bash
# PIC parity tests + both bench_pic workloads (full mode sequence on one context).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pic.py tests/test_gpu_dist.py -q -x 2>&1 | tail -3
for w in uniform c2; do
  timeout 400 python bench_pic.py --workload $w --steps 8 --warmup 2 > gpurun_out/picc_$w.json 2> gpurun_out/picc_$w.err
  tail -2 gpurun_out/picc_$w.err
  python -c "import json; d=json.load(open('gpurun_out/picc_$w.json')); print('$w', {k: (round(v['ms'],3), round(v['frac_of_hbm_peak'],3)) for k, v in d.items() if isinstance(v, dict)})"
done
