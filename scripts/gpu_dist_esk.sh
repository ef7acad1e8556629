#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k "pic" > gpurun_out/de_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/de_pytest.log
