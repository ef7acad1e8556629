#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_ipc.py -x -q > gpurun_out/dist_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/dist_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --force-dist --steps 20 --warmup 5 --no-e2e > gpurun_out/dist1.json 2> gpurun_out/dist1.err; echo "dist rc=$?"; tail -3 gpurun_out/dist1.err; python -c "
import json
for l in open('gpurun_out/dist1.json'):
    if l.startswith('{'): d=json.loads(l); print(d['value'], d['ms_per_step'], d['gpu_launches'])"
