mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench_costs.py --strategies heuristic,timers > gpurun_out/c3t.json 2> gpurun_out/c3t.err; tail -3 gpurun_out/c3t.err; cat gpurun_out/c3t.json
timeout 600 python bench.py --force-dist --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; tail -3 gpurun_out/bench_dist1.err; cat gpurun_out/bench_dist1.json
