#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/gpuclock_diag.py 400 > gpurun_out/r2d_diag.json; echo "diag rc=$?"; cat gpurun_out/r2d_diag.json
timeout 600 python bench_costs.py --steps 30 > gpurun_out/r2d_costs.json 2>gpurun_out/r2d_costs.err; echo "costs rc=$?"; tail -c 2500 gpurun_out/r2d_costs.json; tail -3 gpurun_out/r2d_costs.err
