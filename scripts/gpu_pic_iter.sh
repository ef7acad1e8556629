#!/bin/bash
# PIC iteration: parity tests, bench, launch list, ncu of the push kernel (sorted mode).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pic.py -x -q > gpurun_out/pic_tests.log 2>&1; echo "pic tests rc=$?"; tail -15 gpurun_out/pic_tests.log
timeout 300 python bench_pic.py > gpurun_out/pic.json 2> gpurun_out/pic.err; tail -3 gpurun_out/pic.err; cat gpurun_out/pic.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pic_launches.csv python bench_pic.py --steps 2 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pic_push -s 3 -c 1 -o gpurun_out/prof_pic python bench_pic.py --steps 2 --warmup 2 > gpurun_out/ncu_pic.log 2>&1; tail -1 gpurun_out/ncu_pic.log
