#!/bin/bash
# PIC kernel profile: launch list + one full ncu capture of pic_push_kernel.
mkdir -p gpurun_out
timeout 300 python bench_pic.py > gpurun_out/pic.json 2> gpurun_out/pic.err; tail -3 gpurun_out/pic.err; cat gpurun_out/pic.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pic_launches.csv python bench_pic.py --steps 2 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pic_push -s 2 -c 1 -o gpurun_out/prof_pic python bench_pic.py --steps 1 --warmup 1 > gpurun_out/ncu_pic.log 2>&1; tail -2 gpurun_out/ncu_pic.log
