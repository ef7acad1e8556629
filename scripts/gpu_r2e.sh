#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/gpuclock_fidelity.py > gpurun_out/r2e_gpuclock_native.json; echo "fid rc=$?"; cat gpurun_out/r2e_gpuclock_native.json
timeout 600 python scripts/gpuclock_diag.py 400 > gpurun_out/r2e_diag.json; echo "diag rc=$?"; cat gpurun_out/r2e_diag.json
timeout 900 python -m pytest tests/test_gpu_runs.py tests/test_gpu_kernels.py -q -x > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2e_pytest.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2e_bench.json 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/r2e_bench.json
