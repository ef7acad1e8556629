#!/usr/bin/env python
"""Config C3: cost-strategy sweep on one B200 -- overhead and mapping quality.

Same workload as bench.py (C2 geometry from the kick, 801,499-particle set
tiled R times), balanced over `--ranks` virtual ranks (the LB decisions of an
R-rank job, computed on one GPU).  For each strategy:

  heuristic  uninstrumented fused kernel (counts -> w_p*count + w_c*cells)
  gpuclock   the same kernel instantiated with the clock64 tally
  timers     per-box push launches timed with CUDA events (the paper's
             CUPTI-style strategy): box-sort + one launch per box
  cupti      the same per-box launches timed by CUPTI kernel activity
             records (the paper's actual mechanism)
  measured   the reference's simulated timer (true work x PCG64 jitter)

Reported per strategy: mean fused-kernel time (CUDA events around each
launch), overhead vs the uninstrumented kernel, mean LB efficiency of the
mappings the strategy chose evaluated under TRUE work, adoptions, and (for
gpuclock) Spearman rank correlation of the clock costs with true work.
Prints one JSON object.
"""

from __future__ import annotations

import argparse
import json
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def spearman(a, b):
    ra = np.argsort(np.argsort(a, kind="stable"), kind="stable").astype(float)
    rb = np.argsort(np.argsort(b, kind="stable"), kind="stable").astype(float)
    return float(np.corrcoef(ra, rb)[0, 1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replicas", type=int, default=128)
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--strategies", default="heuristic,gpuclock,timers,cupti,measured")
    args = ap.parse_args()

    import torch

    import bench
    from paper_2104_11385_b200.balancer import efficiency
    from paper_2104_11385_b200.cost import CostVector
    from paper_2104_11385_b200.decomposition import DistributionMapping
    from paper_2104_11385_b200.workload import Simulation, true_work

    dev = torch.device("cuda:0")
    out = {"workload": f"C2 x{args.replicas} replicas, {args.ranks} virtual ranks, "
                       f"{args.steps} steps (first {args.warmup} excluded from timing)",
           "strategies": {}}
    for kind in args.strategies.split(","):
        spec, sc = bench.c2_spec(args.ranks, args.steps, kind)
        sc = replace(sc, initial_mapping="slab")
        pos0, kick0 = bench.base_particles(spec)
        pos = torch.from_numpy(pos0).to(dev).repeat(args.replicas, 1)
        kick = torch.from_numpy(kick0).to(dev).repeat(args.replicas, 1)
        sim = Simulation(sc, spec.policy, spec.build_provider(), device=dev, positions=pos,
                         kick=kick, record_counts=True, time_kernels=True)
        del pos, kick
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sim.run(0, args.warmup)
        torch.cuda.synchronize()
        ev0.record()
        sim.run(args.warmup, args.steps)
        ev1.record()
        torch.cuda.synchronize()
        step_ms = ev0.elapsed_time(ev1) / (args.steps - args.warmup)
        res = sim.result()
        kms = res.kernel_ms[args.warmup:]
        owner = res.initial_owner.copy()
        snaps = dict(res.adoption_snapshots)
        e_true = []
        rho = []
        for s in range(len(res.metrics)):
            if s in snaps:
                owner = snaps[s]
            work = true_work(res.count_trace[s], sc)
            e_true.append(efficiency(CostVector(values=work),
                                     DistributionMapping(owner=owner, n_ranks=args.ranks)))
            if kind in ("gpuclock", "timers", "cupti") and s % 10 == 0:
                occ = res.count_trace[s] > 0
                rho.append(spearman(res.cost_trace[s][occ], work[occ]))
        entry = {"step_ms_mean": step_ms,
                 "kernel_ms_mean": float(np.mean(kms)), "kernel_ms_min": float(np.min(kms)),
                 "mean_eff_true_work": float(np.mean(e_true)),
                 "mean_eff_own_costs": res.summary["mean_efficiency"],
                 "e_true_first": float(e_true[0]), "adoptions": res.summary["adoption_count"],
                 "particles": int(sim.n_init)}
        if rho:
            entry["spearman_vs_true_work_min"] = float(np.min(rho))
            entry["spearman_vs_true_work_mean"] = float(np.mean(rho))
        out["strategies"][kind] = entry
        sim.close()
        del sim
        torch.cuda.empty_cache()
    st = out["strategies"]
    if "heuristic" in st and "gpuclock" in st:
        out["gpuclock_overhead"] = st["gpuclock"]["kernel_ms_mean"] / st["heuristic"]["kernel_ms_mean"] - 1
        out["gpuclock_step_overhead"] = st["gpuclock"]["step_ms_mean"] / st["heuristic"]["step_ms_mean"] - 1
    if "heuristic" in st and "timers" in st:
        out["timers_step_overhead"] = st["timers"]["step_ms_mean"] / st["heuristic"]["step_ms_mean"] - 1
    if "heuristic" in st and "cupti" in st:
        out["cupti_step_overhead"] = st["cupti"]["step_ms_mean"] / st["heuristic"]["step_ms_mean"] - 1
    print(json.dumps(out))


if __name__ == "__main__":
    main()
