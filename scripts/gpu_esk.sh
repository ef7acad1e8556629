#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic_esirkepov.py -q -x 2>&1 | tail -3
timeout 600 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast_resort,push_deposit_esk1,push_deposit_esk3,push_deposit_esk3_resort,full_step_esk3_resort > gpurun_out/esk_c2.json 2>&1; echo "c2 rc=$?"; tail -c 2500 gpurun_out/esk_c2.json
timeout 600 python bench_pic.py --workload uniform --steps 6 --warmup 2 --resort 10 --modes push_deposit_esk1,push_deposit_esk3 > gpurun_out/esk_uni.json 2>&1; echo "uni rc=$?"; tail -c 1500 gpurun_out/esk_uni.json
timeout 800 ncu --set full --import-source on --clock-control none -k regex:pic_esk_kernel -s 1 -c 1 -o gpurun_out/esk3_full python bench_pic.py --steps 1 --warmup 1 --modes push_deposit_esk3_resort > gpurun_out/esk3_full.log 2>&1; echo "ncu rc=$?"
