#!/usr/bin/env python
"""Config C5: no LB vs static LB vs dynamic LB speedup, against the
performance-model maximum S_max = (1/E0)^x (perfmodel.py).

Scenario: the C2 geometry with the high-imbalance blob of SURVEY 7 (centre
[60, 480], core 44: the blob sits inside one rank's slab, E0 ~ 0.2 at 8
ranks) from the kick on, the 801,499-particle-class set tiled R times, slab
initial mapping, knapsack remaps with GpuClock costs.  Policies:
  none     no rebalancing (slab mapping throughout)
  static   one knapsack attempt at step 0
  dynamic  knapsack attempt every 10 steps (10 % relative threshold)

Mode (one GPU is available this round): `python bench_lb.py --emulate R`
runs R ranks as threads through the full multi-GPU code path (exchange
kernels, replicated LB, adoption-time migration).  Each rank's fused step
kernel runs alone (a lock serializes them) and is timed with CUDA events
recorded by libLBX immediately around its launch; the emulated step time is
the MAX over ranks of those times (the compute-imbalance part of an R-GPU
step, measured on B200) plus, on adoption steps, a modelled redistribution
time: max over ranks of the bytes it sends (48-byte records) / 770 GB/s (the
measured NVLink peer bandwidth, B200_PROFILING.md).  On a multi-GPU box the
same path runs for real under torchrun via `bench.py --gpus N`.
Prints one JSON object.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def scenario(ranks, steps, policy, speed=0.035, drift=0.01, strategy="knapsack",
             migration_ratio=0.0):
    from paper_2104_11385_b200.balancer import Strategy
    from paper_2104_11385_b200.scenarios import apply_overrides, load_spec
    from paper_2104_11385_b200.workload import BlobSpec, KickSpec

    spec = apply_overrides(load_spec("default"), cost="gpuclock", ranks=ranks, steps=steps,
                           policy=strategy if policy == "dynamic" else policy)
    if policy != "none":
        spec = replace(spec, policy=replace(spec.policy, strategy=Strategy(strategy),
                                            migration_ratio=migration_ratio))
    sc = replace(spec.scenario, blob=BlobSpec(center=(60.0, 480.0), core_radius=44.0,
                                              edge_scale=4.0, particles_per_cell=55.0),
                 kick=KickSpec(step=0, speed=speed, drift=drift), initial_mapping="slab")
    return spec, sc


def make_timed_engine(lock, log, physics="surrogate"):
    from paper_2104_11385_b200.parallel import DeviceEngine, PicEngine

    if physics == "pic":
        class TimedPic(PicEngine):
            # A rank's step = its particle kernels + its (replicated) current
            # gather / field solve + its emigrant partition.  Each part runs
            # under the lock after a device-wide synchronize, so nothing else
            # is on the GPU (the other ranks are either queued on the lock or
            # parked in the next collective); the cross-rank sums are not timed.
            def local_step(self, wp, wc):
                import torch
                with lock:
                    torch.cuda.synchronize()
                    self.time_step = True
                    super().local_step(wp, wc)
                    log.setdefault(self.rank, []).append(self.last_ms)

            def finish(self):
                import torch
                with lock:
                    torch.cuda.synchronize()
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                    ev[0].record()
                    super().finish()
                    ev[1].record()
                    ev[1].synchronize()
                    log[self.rank][-1] += ev[0].elapsed_time(ev[1])

            def push(self, wp, wc):
                import torch
                self.local_step(wp, wc)
                self.current_sum_finish()   # guard exchange + (timed) finish + field rings
                with lock:
                    torch.cuda.synchronize()
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                    ev[0].record()
                    send_counts, nout = self.partition()
                    ev[1].record()
                    ev[1].synchronize()
                    log[self.rank][-1] += ev[0].elapsed_time(ev[1])
                return self.counts, self.clk, send_counts, nout
        return TimedPic

    class TimedEngine(DeviceEngine):
        def push(self, wp, wc):
            import ctypes as C

            import torch

            from paper_2104_11385_b200 import _lib
            with lock:   # ranks' kernels run one at a time, on an otherwise idle GPU
                torch.cuda.synchronize()
                _lib.lib.lbx_ctx_enable_timing(self.ctx.handle, 1)
                out = super().push(wp, wc)
                ms = C.c_float()
                _lib.check(_lib.lib.lbx_ctx_last_kernel_ms(self.ctx.handle, C.byref(ms)))
                log.setdefault(self.rank, []).append(ms.value)
            return out

    return TimedEngine


def run_emulated(R, steps, replicas, policy, speed=0.035, drift=0.01, strategy="knapsack",
                 migration_ratio=0.0, physics="surrogate", exchange="nccl", shape_order=0,
                 pic_fast=False):
    import torch

    import bench
    from paper_2104_11385_b200.parallel import DistributedSimulation, ThreadComm

    spec, sc = scenario(R, steps, policy, speed, drift, strategy, migration_ratio)
    from paper_2104_11385_b200.workload import kick_velocities, sample_blob
    pos = sample_blob(sc)
    kick = kick_velocities(pos, sc)
    lock, log = threading.Lock(), {}
    shared = ThreadComm.shared(R)
    sims, errs = [None] * R, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            torch.cuda.set_stream(torch.cuda.Stream())   # per-rank stream (thread-local)
            sim = DistributedSimulation(sc, spec.policy, spec.build_provider(),
                                        comm=ThreadComm(shared, r),
                                        engine_factory=make_timed_engine(lock, log, physics),
                                        positions=pos, kick=kick, device="cuda:0",
                                        replicas=replicas,
                                        capacity=pos.shape[0] * replicas + 4096,
                                        physics=physics, exchange=exchange,
                                        pic={"shape_order": shape_order, "resort": 10,
                                             "fast": pic_fast}
                                        if physics == "pic" else None,
                                        pipeline=False)   # ranks' pushes timed one by one
            sim.run()
            sims[r] = sim
        except Exception as e:
            errs.append(e)
            shared["bar"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    per_step = np.max(np.array([log[r] for r in range(R)]), axis=0)   # [steps]
    # adoption-time redistribution over NVLink, modelled: each rank sends its
    # lost boxes' particles (48-byte records); the step pays the slowest rank
    # at the measured 770 GB/s per-direction peer bandwidth (B200_PROFILING.md)
    sent = np.array([s.moved[:len(per_step)] for s in sims])            # [R, steps]
    migrate_ms = sent.max(axis=0) * 48 / 770e9 * 1e3
    res = sims[0].result()
    moved = int(sent.sum())
    for s in sims:
        s.close(collective=False)   # every rank thread has finished
    return per_step, migrate_ms, res, moved, pos.shape[0] * replicas


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--emulate", type=int, default=0, help="ranks emulated on one GPU")
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--replicas", type=int, default=128)
    ap.add_argument("--warmup-steps", type=int, default=1)
    ap.add_argument("--speed", type=float, default=0.035, help="kick speed (cells/step)")
    ap.add_argument("--drift", type=float, default=0.01, help="axial drift (cells/step)")
    ap.add_argument("--strategy", default="knapsack", choices=["knapsack", "sfc"])
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="emigrant exchange of the emulated ranks (p2p: fused peer writes)")
    ap.add_argument("--physics", default="surrogate", choices=["surrogate", "pic"],
                    help="pic: the 2D3V PIC step (pic.py) per rank (its particles cell-sorted "
                         "every 10 steps), GpuClock from its kernel, guard-cell current / "
                         "field exchange over off-rank faces")
    ap.add_argument("--shape-order", type=int, default=0, choices=[0, 1, 2, 3],
                    help="pic: 0 = CIC deposit, 1-3 = charge-conserving Esirkepov deposit "
                         "with that B-spline order (the paper's 3) -- its GpuClock tally "
                         "drives the remap")
    ap.add_argument("--pic-fast", action="store_true",
                    help="pic with shape order 0: tolerance mode (LBX_PIC_FAST)")
    ap.add_argument("--migration-ratio", type=float, default=0.0,
                    help=">0: migration-aware adoption gate (pushes per moved particle)")
    args = ap.parse_args()
    if not args.emulate:
        raise SystemExit("multi-GPU mode: run under torchrun with bench.py --gpus N for the "
                         "throughput line; this script's LB comparison uses --emulate R here")
    from paper_2104_11385_b200.perfmodel import EXPONENT_PRESETS, achieved_fraction, max_speedup

    R = args.emulate
    out = {"mode": f"EMULATED {R} ranks on one B200 (per-rank kernels timed alone; "
                   "step time = max over ranks; migration modelled at NVLink rates) -- a "
                   "model, not a multi-GPU measurement", "ranks": R, "steps": args.steps,
           "kick": {"speed": args.speed, "drift": args.drift}, "strategy": args.strategy,
           "migration_ratio": args.migration_ratio, "physics": args.physics,
           "shape_order": args.shape_order, "pic_fast": args.pic_fast,
           "warmup_steps_dropped": args.warmup_steps, "policies": {}}
    w = args.warmup_steps
    for policy in ("none", "static", "dynamic"):
        per_step, mig, res, moved, n = run_emulated(R, args.steps, args.replicas, policy,
                                                    args.speed, args.drift, args.strategy,
                                                    args.migration_ratio, args.physics,
                                                    args.exchange, args.shape_order,
                                                    args.pic_fast)
        effs = [m.efficiency_after for m in res.metrics]
        # speedups use the raw (unclipped) step times; only the compute of
        # the first `w` steps (lazy allocations, graph capture) is dropped,
        # the same rule for every policy -- their modelled migration (the
        # step-0 adoption of static / dynamic) is always counted
        med = float(np.median(per_step[w:])) if len(per_step) > w else 0.0
        total = per_step + mig
        out["policies"][policy] = {
            "time_ms": float(per_step[w:].sum() + mig.sum()),
            "compute_ms": float(per_step[w:].sum()),
            "median_step_ms": med,
            "migration_ms_modelled": float(mig.sum()),
            "ms_per_step": float((per_step[w:].sum() + mig.sum()) / max(1, len(per_step) - w)),
            "e0": float(res.metrics[0].efficiency_before), "mean_eff": float(np.mean(effs)),
            "adoptions": res.summary["adoption_count"], "particles_migrated": moved,
            "particles": n, "step_ms": [round(float(t), 4) for t in total]}
    P = out["policies"]
    x = EXPONENT_PRESETS["2d3v"]
    e0 = P["none"]["e0"]
    s_max = max_speedup(e0, x)
    out["speedup_dynamic_vs_none"] = P["none"]["time_ms"] / P["dynamic"]["time_ms"]
    out["speedup_static_vs_none"] = P["none"]["time_ms"] / P["static"]["time_ms"]
    out["speedup_dynamic_vs_static"] = P["static"]["time_ms"] / P["dynamic"]["time_ms"]
    out["model"] = {"E0": e0, "x": x, "S_max": s_max,
                    "achieved_fraction": achieved_fraction(out["speedup_dynamic_vs_none"], s_max)}
    print(json.dumps(out))


if __name__ == "__main__":
    if os.environ.get("LBX_DEBUG_HANG"):      # dump every thread's stack if stuck
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["LBX_DEBUG_HANG"]), exit=True)
    main()
