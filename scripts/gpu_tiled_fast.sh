#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic_fast.py tests/test_gpu_pic.py -q -x > gpurun_out/tf_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tf_pytest.log
timeout 900 python bench_pic.py --workload uniform --steps 10 --warmup 2 --resort 10 --modes push_deposit_tiled,push_deposit_fast_tiled > gpurun_out/tf_bench.json 2>&1; echo "bench rc=$?"; tail -c 900 gpurun_out/tf_bench.json; echo
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pic_tile_kernel -c 1 -o gpurun_out/tf_full python bench_pic.py --workload uniform --steps 1 --warmup 0 --modes push_deposit_fast_tiled > gpurun_out/tf_full.log 2>&1; echo "ncu rc=$?"
