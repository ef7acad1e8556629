#!/bin/bash
# Round-2 end-of-session verification: all GPU tests, smoke, bench (both
# arms), NCCL self-launch path at N=1, launch list + full ncu capture of the
# headline kernel.  Outputs -> gpurun_out/r2h_*
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2h_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2h_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2h_smoke.log
timeout 900 python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo "bench rc=$?"; grep '^{' gpurun_out/r2h_bench.json | tail -1 | head -c 700; echo
timeout 900 python bench.py --impl reference > gpurun_out/r2h_bench_ref.json 2> gpurun_out/r2h_bench_ref.err; echo "ref rc=$?"; grep '^{' gpurun_out/r2h_bench_ref.json | tail -1 | head -c 300; echo
timeout 600 python bench.py --gpus 1 --force-dist --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2h_force_dist.log 2>&1; echo "force-dist rc=$?"; grep -ci "nranks" gpurun_out/r2h_force_dist.log; grep '^{' gpurun_out/r2h_force_dist.log | tail -1 | head -c 400; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2h_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-native --no-pic > gpurun_out/r2h_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 1 -c 1 -o gpurun_out/r2h_stream_full python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-native --no-pic > gpurun_out/r2h_stream_full.log 2>&1; echo "ncu full rc=$?"
