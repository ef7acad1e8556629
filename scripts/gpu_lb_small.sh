#!/bin/bash
mkdir -p gpurun_out
for ex in nccl p2p; do
  t0=$(date +%s); timeout 240 python bench_lb.py --emulate 8 --replicas 4 --steps 20 --speed 0.3 --drift 0.3 --exchange $ex > gpurun_out/lbs_$ex.json 2> gpurun_out/lbs_$ex.err; echo "$ex rc=$? $(( $(date +%s) - t0 )) s"; tail -2 gpurun_out/lbs_$ex.err; head -c 300 gpurun_out/lbs_$ex.json; echo
done
