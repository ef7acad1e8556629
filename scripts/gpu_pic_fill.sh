#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pic.py tests/test_gpu_dist.py -x -q > gpurun_out/pic_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pic_tests.log
for w in uniform c2; do
timeout 600 python bench_pic.py --workload $w --steps 6 --warmup 2 > gpurun_out/pic_$w.json 2> gpurun_out/pic_$w.err; echo "pic $w rc=$?"; tail -2 gpurun_out/pic_$w.err; python -c "
import json; d=json.load(open('gpurun_out/pic_$w.json')); print({k:(round(d[k]['ms'],2), round(d[k]['frac_of_hbm_peak'],3), d[k]['ms_per_step']) for k in ('push_deposit','push_deposit_inplace','full_step')})"
done
