mkdir -p gpurun_out
python bench_pic.py > gpurun_out/pic.json 2> gpurun_out/pic.err; tail -3 gpurun_out/pic.err; cat gpurun_out/pic.json
timeout 500 ncu --set full --clock-control none --import-source on -k regex:pic_push -s 2 -c 1 -o gpurun_out/prof_pic python bench_pic.py --steps 1 --warmup 1 > gpurun_out/ncu_pic.log 2>&1; tail -2 gpurun_out/ncu_pic.log
