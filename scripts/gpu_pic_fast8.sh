#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic_fast.py tests/test_gpu_pic.py -q -x > gpurun_out/pf8_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pf8_pytest.log
timeout 900 python bench_pic.py --steps 10 --warmup 3 --resort 10 --modes push_deposit_fast,push_deposit_fast_resort,push_deposit_resort > gpurun_out/pf8_c2.json 2>&1; echo "c2 rc=$?"; tail -c 1500 gpurun_out/pf8_c2.json; echo
