#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic.py tests/test_gpu_pic_fast.py -q -x > gpurun_out/s2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s2_pytest.log
bash scripts/gpu_sort_prof.sh 2>&1 | grep -E "pic_count|pic_sort_scatter|gpu__time|dram__bytes" | head -12
timeout 900 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast_resort > gpurun_out/s2_c2.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/s2_c2.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print(k, round(v['ms'],3), round(v['ms_pipelined'],3), v['ms_per_step'])"
