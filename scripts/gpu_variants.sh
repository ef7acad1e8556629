#!/bin/bash
# A/B the PIC build variants: bench_pic per libLBX.<v>.so (MODES / WORKLOAD / STEPS env)
mkdir -p gpurun_out
for rep in 1 2; do
for v in "$@"; do
  LBX_VARIANT=$v timeout 300 python bench_pic.py --workload ${WORKLOAD:-c2} --steps ${STEPS:-8} --warmup 2 \
    --modes ${MODES:-push_deposit,push_deposit_inplace} > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.load(open(f"gpurun_out/var_{v}.json"))
print(v, {k: round(x["ms"], 3) for k, x in d.items() if isinstance(x, dict)})
PY
done
done
