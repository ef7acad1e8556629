#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_3d.py -q -x > gpurun_out/3d_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/3d_pytest.log
for v in "" m4; do
LBX_VARIANT=$v timeout 600 python bench_3d.py > gpurun_out/3d_$v.json 2>&1; echo "$v rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/3d_$v.json').read().strip().splitlines()[-1]); print('$v', {k: d[k] for k in d if not isinstance(d[k], (dict, list))}); print(d.get('roofline'))" 2>&1 | head -4
done
