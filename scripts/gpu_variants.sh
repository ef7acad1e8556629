#!/bin/bash
# A/B the PIC build variants: bench_pic per libLBX.<v>.so
mkdir -p gpurun_out
for v in "$@"; do
  LBX_VARIANT=$v timeout 300 python bench_pic.py --steps 8 --warmup 2 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.load(open(f"gpurun_out/var_{v}.json"))
print(v, {k: round(d[k]["ms"], 3) for k in ("push_deposit", "push_deposit_inplace", "full_step")},
      d["push_deposit_inplace"]["ms_per_step"])
PY
done
