#!/bin/bash
mkdir -p gpurun_out
LBX_DEBUG_HANG=60 timeout 200 python bench_lb.py --emulate 2 --replicas 1 --steps 6 --speed 0.3 --drift 0.3 --exchange p2p > gpurun_out/lbd.json 2> gpurun_out/lbd.err; echo rc=$?; grep -v "^  File \"/opt" gpurun_out/lbd.err | head -90
