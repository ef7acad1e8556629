python -m pytest tests/test_gpu_3d.py -x -q 2>&1 | tail -2
python bench_3d.py > gpurun_out/c4.json 2> gpurun_out/c4.err; tail -3 gpurun_out/c4.err; cat gpurun_out/c4.json
timeout 900 python bench_lb.py --emulate 8 --speed 0.3 --drift 0.3 --steps 120 > gpurun_out/lb8b.json 2> gpurun_out/lb8b.err; tail -5 gpurun_out/lb8b.err; cat gpurun_out/lb8b.json
timeout 500 ncu --set full --clock-control none --import-source on -k regex:pic_push -s 2 -c 1 -o gpurun_out/prof_pic3 python bench_pic.py --steps 1 --warmup 1 > gpurun_out/ncu_pic.log 2>&1; tail -1 gpurun_out/ncu_pic.log
