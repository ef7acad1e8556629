#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_runs.py -q -x -k "long_run" > gpurun_out/long_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/long_pytest.log
