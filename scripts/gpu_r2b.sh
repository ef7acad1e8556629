#!/bin/bash
mkdir -p gpurun_out
env | grep -i nccl
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_runs.py tests/test_gpu_cli.py tests/test_gpu_pic.py -q -x -k "not pic or gpuclock" > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2b_pytest.log
timeout 600 python scripts/gpuclock_fidelity.py > gpurun_out/r2b_gpuclock_native.json; echo "fid rc=$?"; cat gpurun_out/r2b_gpuclock_native.json
timeout 300 python bench.py --gpus 1 --force-dist --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2b_force.log 2>&1; echo "force rc=$?"; grep -i "nranks\|NCCL" gpurun_out/r2b_force.log | head; tail -c 600 gpurun_out/r2b_force.log
