#!/bin/bash
# Esirkepov kernel: tests, C2 bench (orders 1 and 3), ncu of order 3. $1 = output tag
T=${1:-esk}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic_esirkepov.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
timeout 900 python bench_pic.py --steps 6 --warmup 2 --resort 10 --modes push_deposit_esk1,push_deposit_esk3,push_deposit_esk3_resort > gpurun_out/${T}_c2.json 2>&1; echo "c2 rc=$?"; tail -c 1200 gpurun_out/${T}_c2.json; echo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pic_esk_kernel -c 1 -o gpurun_out/${T}_full python bench_pic.py --steps 1 --warmup 0 --modes push_deposit_esk3_resort > gpurun_out/${T}_full.log 2>&1; echo "ncu full rc=$?"
