#!/usr/bin/env python
"""Config C4: 3D blob, 256 boxes, SFC vs knapsack (parity unpinned: the
reference is 2D only).

Workload: 256 x 256 x 128 cells, 32-cell boxes (8 x 8 x 4 = 256 boxes), a
spherical blob (centre (128, 128, 64), core 40, skirt 4, 2 particles/cell,
seed 1) from the kick (radial 0.035 + drift 0.01), tiled R times (default
140 -> ~1e8 particles), GpuClock costs.  Measured on one B200:
  * fused 3D step throughput (particle-pushes/s) and HBM roofline
    (72 B/particle: read z,y,x,vz,vy,vx, write z,y,x);
  * for R = 1, 2, 4, 8 ranks and each strategy (knapsack, SFC): the LB
    efficiency of the proposed mapping on the measured GpuClock costs AND
    under true work, the number of off-rank box faces (SFC's locality
    advantage), and the modelled R-GPU step time = measured 1-GPU step x
    (max rank work / total work) -- a strong-scaling estimate, labelled as
    such (one GPU is available this round).
Prints one JSON object.

`--distributed` (under torchrun, one rank per GPU, NCCL): the real
multi-GPU path instead -- three_d.Distributed3D with the scenario's
particles split by box ownership (strong scaling: the total is fixed), the
fused 3D exchange push, all-reduced counts, record all-to-all, replicated
LB and adoption-time migration; device-timed (CUDA events, barrier, max
over ranks) pushes/s of the whole job.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replicas", type=int, default=140)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--distributed", action="store_true",
                    help="real multi-GPU run (torchrun, NCCL): Distributed3D strong scaling")
    ap.add_argument("--strategy", default="knapsack", choices=["knapsack", "sfc"])
    ap.add_argument("--interval", type=int, default=10)
    args = ap.parse_args()
    if args.distributed:
        return distributed_main(args)

    import torch

    import bench
    from paper_2104_11385_b200.balancer import BalancePolicy, efficiency, knapsack_assign, sfc_assign
    from paper_2104_11385_b200.cost import CostVector, make_provider
    from paper_2104_11385_b200.decomposition import DistributionMapping, morton_order_3d
    from paper_2104_11385_b200.three_d import (Scenario3D, Simulation3D, kick_velocities_3d,
                                               sample_blob_3d)

    total = args.warmup + args.steps
    cfg = Scenario3D("c4-3d-blob", (256, 256, 128), 32, 1, (128.0, 128.0, 64.0), 40.0, 4.0,
                     2.0, kick_step=0, kick_speed=0.035, kick_drift=0.01, total_steps=total)
    pos0 = sample_blob_3d(cfg)
    kick0 = kick_velocities_3d(pos0, cfg)
    R = args.replicas
    dev = torch.device("cuda:0")
    pos = torch.from_numpy(pos0).to(dev).repeat(R, 1)
    kick = torch.from_numpy(kick0).to(dev).repeat(R, 1)
    sim = Simulation3D(cfg, BalancePolicy(interval=total + 1), make_provider("gpuclock"),
                       device=dev, positions=pos, kick=kick, record_counts=True,
                       stable_order=False)
    del pos, kick
    n = sim.n_init
    sim.run(0, args.warmup)
    torch.cuda.synchronize()
    import ctypes as C

    from paper_2104_11385_b200 import _lib
    ms, kms = [], []
    stream = torch.cuda.current_stream(dev)
    _lib.lib.lbx_ctx_enable_timing(sim.ctx.handle, 1)
    for s in range(args.warmup, total):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.run(s, s + 1)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        k = C.c_float()
        _lib.lib.lbx_ctx_last_kernel_ms(sim.ctx.handle, C.byref(k))
        kms.append(k.value)
    step_ms = float(np.mean(ms))
    kernel_ms = float(np.mean(kms))
    peak, peak_src = bench.peaks()
    achieved = 72 * n / (step_ms / 1e3) / 1e9
    counts = sim.out["count_trace"][total - 1]
    clk = sim.out["cost_trace"][total - 1]
    work = cfg.work_weights[0] * counts + cfg.work_weights[1] * 32 ** 3
    curve = morton_order_3d(cfg.grid)
    g = cfg.grid
    ids = np.arange(cfg.n_boxes).reshape(g)
    fa = np.concatenate([ids[:-1].ravel(), ids[:, :-1].ravel(), ids[:, :, :-1].ravel()])
    fb = np.concatenate([ids[1:].ravel(), ids[:, 1:].ravel(), ids[:, :, 1:].ravel()])
    # measured per-rank step times: every rank's particles (the boxes the
    # mapping gives it) pushed by the fused 3D kernel alone on the GPU, timed
    # with CUDA events around the launch; R-rank step = max over ranks
    n_now = int(sim.n)
    st = {k: sim.arr[k][:n_now] for k in ("z", "y", "x", "vz", "vy", "vx")}
    M = cfg.box_size
    box_of = ((st["z"] / M).long() * g[1] + (st["y"] / M).long()) * g[2] + (st["x"] / M).long()
    rcfg = Scenario3D("c4-rank", cfg.domain_extent, M, 1, cfg.center, cfg.core_radius,
                      cfg.edge_scale, cfg.particles_per_cell, kick_step=0, kick_speed=0.0,
                      kick_drift=0.0, total_steps=4)

    def rank_kernel_ms(mask):
        idx = torch.nonzero(mask).squeeze(1)
        if idx.numel() == 0:
            return 0.0
        p = torch.stack([st[k].index_select(0, idx) for k in ("z", "y", "x")], 1)
        v = torch.stack([st[k].index_select(0, idx) for k in ("vz", "vy", "vx")], 1)
        rs = Simulation3D(rcfg, BalancePolicy(interval=99), make_provider("gpuclock"),
                          device=dev, positions=p, kick=v, stable_order=False)
        del p, v
        rs.run(0, 2)
        _lib.lib.lbx_ctx_enable_timing(rs.ctx.handle, 1)
        t = []
        for s_ in (2, 3):
            rs.run(s_, s_ + 1)
            k = C.c_float()
            _lib.lib.lbx_ctx_last_kernel_ms(rs.ctx.handle, C.byref(k))
            t.append(k.value)
        rs.close()
        torch.cuda.empty_cache()
        return float(np.mean(t))

    t1 = rank_kernel_ms(torch.ones(n_now, dtype=torch.bool, device=dev))
    scaling = {}
    for r in (1, 2, 4, 8):
        row = {}
        for name in ("knapsack", "sfc"):
            cv = CostVector(values=clk)
            own = (knapsack_assign(cv, r).owner if name == "knapsack"
                   else sfc_assign(cv, curve, r).owner)
            dm = DistributionMapping(owner=own, n_ranks=r)
            e_clk = efficiency(cv, dm)
            e_true = efficiency(CostVector(values=work), dm)
            loads = np.bincount(own, weights=work, minlength=r)
            own_t = torch.as_tensor(np.array(own), device=dev)[box_of]
            per_rank = [rank_kernel_ms(own_t == q) for q in range(r)]
            row[name] = {"eff_gpuclock": e_clk, "eff_true_work": e_true,
                         "offrank_faces": int((own[fa] != own[fb]).sum()),
                         "measured_rank_kernel_ms": per_rank,
                         "measured_step_ms": max(per_rank),
                         "measured_speedup": t1 / max(per_rank),
                         "model_step_ms": step_ms * loads.max() / loads.sum(),
                         "model_speedup": float(loads.sum() / loads.max())}
        scaling[str(r)] = row
    out = {"workload": f"3D blob 256x256x128 cells, 256 boxes (8x8x4), {n} particles "
                       f"({len(pos0)} x {R} replicas), GpuClock", "particles": n,
           "step_ms": step_ms, "pushes_per_s": n / (step_ms / 1e3),
           "kernel_ms": kernel_ms,
           "roofline": {"bytes_per_particle": 72,
                        "achieved_gbs": 72 * n / (kernel_ms / 1e3) / 1e9, "peak_gbs": peak,
                        "frac": 72 * n / (kernel_ms / 1e3) / 1e9 / peak, "peak_source": peak_src,
                        "note": "fused 3D kernel, CUDA events around its launch"},
           "whole_step_gbs": achieved,
           "compaction": "O(removed) hole filling (stable_order=False)",
           "strategies_by_ranks": scaling,
           "kernel_ms_all_particles_1rank": t1,
           "note": "measured_*: each rank's particle share pushed alone by the fused 3D kernel "
                   "on the B200 (CUDA events), R-rank step = max over ranks, exchange not "
                   "included; model_*: 1-GPU step x max rank work share"}
    sim.close()
    print(json.dumps(out))


def distributed_main(args):
    """Config C4 on WORLD_SIZE GPUs through Distributed3D (see module doc)."""
    import os
    import time

    import torch
    import torch.distributed as dist

    from paper_2104_11385_b200.balancer import BalancePolicy, Strategy
    from paper_2104_11385_b200.cost import make_provider
    from paper_2104_11385_b200.parallel import TorchComm
    from paper_2104_11385_b200.three_d import (Distributed3D, Scenario3D, kick_velocities_3d,
                                               sample_blob_3d)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    total = args.warmup + args.steps
    cfg = Scenario3D("c4-3d-blob", (256, 256, 128), 32, world, (128.0, 128.0, 64.0), 40.0, 4.0,
                     2.0, kick_step=0, kick_speed=0.035, kick_drift=0.01, total_steps=total,
                     initial_mapping="sfc" if args.strategy == "sfc" else "knapsack")
    pos0 = sample_blob_3d(cfg)
    kick0 = kick_velocities_3d(pos0, cfg)
    pol = BalancePolicy(strategy=Strategy(args.strategy), interval=args.interval)
    sim = Distributed3D(cfg, pol, make_provider("gpuclock"), comm=TorchComm(), device=dev,
                        positions=pos0, kick=kick0, replicas=args.replicas,
                        capacity=int(len(pos0) * args.replicas * min(1.0, 2.5 / world)) + 4096)
    sim.run(0, args.warmup)
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    sim.run(args.warmup, total)
    e1.record()
    torch.cuda.synchronize(dev)
    dist.barrier()
    wall = time.perf_counter() - t0
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    n_total = sim.n_total
    if rank == 0:
        print(json.dumps({
            "workload": "C4 3D blob 256x256x128, 256 boxes, GpuClock, "
                        f"{args.strategy} every {args.interval} (Distributed3D)",
            "n_gpus": world, "particles": n_total, "steps": args.steps,
            "ms_per_step": float(ms.item()) / args.steps,
            "pushes_per_s": n_total * args.steps / (float(ms.item()) / 1e3),
            "wall_s": wall, "scaling": "strong", "adoptions": int(sim.souts.n_adoptions),
            "emigrated_per_step": float(sim.emigrated[args.warmup:total].mean()),
            "migrated": int(sim.moved.sum())}), flush=True)
    sim.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
