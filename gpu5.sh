mkdir -p gpurun_out
python -m pytest tests/test_gpu_cli.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --force-dist --steps 10 --warmup 3 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; tail -5 gpurun_out/bench_dist1.err; cat gpurun_out/bench_dist1.json
timeout 600 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --force-dist --steps 10 --warmup 3 --replicas 64 2>&1 | tail -2
python bench.py --impl reference --cpu-seconds 8 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -3 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
