#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench_pic.py --workload uniform --steps 10 --warmup 2 --resort 10 --modes push_deposit_tiled,push_deposit_fast > gpurun_out/tu_bench.json 2>&1; echo "bench rc=$?"; tail -c 900 gpurun_out/tu_bench.json; echo
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pic_tile_kernel -c 1 -o gpurun_out/tu_full python bench_pic.py --workload uniform --steps 1 --warmup 0 --modes push_deposit_tiled > gpurun_out/tu_full.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tu_launches.csv python bench_pic.py --workload uniform --steps 2 --warmup 0 --resort 10 --modes push_deposit_tiled > gpurun_out/tu_launches.log 2>&1; echo "launches rc=$?"
