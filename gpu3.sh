mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|Socket|Core|Thread" | head -5
python bench_costs.py > gpurun_out/c3.json 2> gpurun_out/c3.err; tail -3 gpurun_out/c3.err; cat gpurun_out/c3.json
timeout 400 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 4 -c 1 -o gpurun_out/prof_stream python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
ls -la gpurun_out
