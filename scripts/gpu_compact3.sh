#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/cp3_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/cp3_pytest.log
