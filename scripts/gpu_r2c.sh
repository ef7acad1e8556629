#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/gpuclock_fidelity.py > gpurun_out/r2c_gpuclock_native.json; echo "fid rc=$?"; cat gpurun_out/r2c_gpuclock_native.json
timeout 900 python -m pytest tests/test_gpu_runs.py -q -x -k "gpuclock" > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2c_pytest.log
timeout 600 python bench_costs.py > gpurun_out/r2c_costs.json 2>gpurun_out/r2c_costs.err; echo "costs rc=$?"; tail -c 2500 gpurun_out/r2c_costs.json
