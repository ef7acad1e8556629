#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python bench_costs.py > gpurun_out/r2h_c3.json 2> gpurun_out/r2h_c3.err; echo "c3 rc=$?"; tail -c 1500 gpurun_out/r2h_c3.json
