#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/kern_tests.log 2>&1; echo "kernel tests rc=$?"; tail -3 gpurun_out/kern_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e'])"
