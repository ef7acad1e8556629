python -m pytest tests/test_gpu_pic.py -x -q 2>&1 | tail -3
python bench_pic.py > gpurun_out/pic.json 2> gpurun_out/pic.err; tail -3 gpurun_out/pic.err; cat gpurun_out/pic.json
for sp in "0.035 0.01 60" "0.15 0.15 120" "0.3 0.3 120"; do set -- $sp; timeout 900 python bench_lb.py --emulate 8 --speed $1 --drift $2 --steps $3 > gpurun_out/lb8_$1.json 2> gpurun_out/lb8_$1.err; tail -2 gpurun_out/lb8_$1.err; cat gpurun_out/lb8_$1.json; done
