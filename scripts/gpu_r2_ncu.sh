#!/bin/bash
# launch list + full ncu capture of the headline kernel (no resident-kernel lines under ncu)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-native --no-pic > gpurun_out/r2f_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 1 -c 1 -o gpurun_out/r2f_stream_full python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-native --no-pic > gpurun_out/r2f_stream_full.log 2>&1; echo "ncu full rc=$?"
