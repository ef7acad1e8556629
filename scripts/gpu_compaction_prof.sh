#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/compaction_probe.py 3 > gpurun_out/cp_bench.json 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/cp_bench.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cp_launches.csv python scripts/compaction_probe.py 2 > gpurun_out/cp_launches.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 -o gpurun_out/cp_full python scripts/compaction_probe.py 2 > gpurun_out/cp_full.log 2>&1; echo "ncu full rc=$?"
