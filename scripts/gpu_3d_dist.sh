#!/bin/bash
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench_3d.py --distributed --steps 6 --warmup 2 > gpurun_out/3d_dist.json 2> gpurun_out/3d_dist.err; echo rc=$?; tail -3 gpurun_out/3d_dist.err; tail -c 800 gpurun_out/3d_dist.json
