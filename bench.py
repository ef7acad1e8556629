#!/usr/bin/env python
"""Benchmark: particle-pushes/s including in-situ cost assessment, plus LB
efficiency, on B200 (BASELINE.json metric; workload = config C2).

Workload (config C2, "2D laser-ion dense-slab target, GpuClock costs,
dynamic LB every 10 steps"): the reference's default.yaml geometry -- 960x960
cells, 32-cell boxes (900 boxes), dense blob (core 64, skirt 4, 55 ppc)
sampled with the reference's own PCG64 stream -- from the kick step onward
(radial kick, speed 0.035, drift 0.01), GpuClock costs, knapsack remap
attempted every 10 steps with a 10% relative threshold.  To fill a B200 the
801,499-particle set is tiled R times (default R=128 -> 102.6 M particles,
3.3 GB of particle state): every replica evolves identically, so per-box
counts are exactly R x the reference's (checked by tests/test_gpu_bench_parity).

One step = the fused sm_100a kernel (push + absorb + stable compaction +
per-box counts + heuristic cost + GpuClock tally) + the step record written
to mapped host memory + the native host loop (cost vector, efficiency,
knapsack attempt every 10 steps).  Inputs (3.3 GB) are larger than L2
(126 MB), so no flush is needed between steps.

--impl reference: the reference's own CPU implementation (its compiled
Cython kernels from oracle/_ref, with the oracle port of its numpy cost and
balancer code) on the same workload, one process per host core, each on a
bounded sample; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-pushes/s incl. in-situ cost assessment; LB efficiency at 1-8 B200"
UNIT = "particle-pushes/s"
BYTES_PER_PUSH = 48  # read z,x,vz,vx + write z,x (fp64), SURVEY 8(d)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="lbx", choices=["lbx", "reference"])
    ap.add_argument("--replicas", type=int, default=128)
    ap.add_argument("--cost", default="gpuclock")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the multi-GPU box-ownership path even at N=1 (testing)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def c2_spec(n_ranks: int, steps: int, cost: str):
    from dataclasses import replace

    from paper_2104_11385_b200.scenarios import apply_overrides, load_spec

    spec = apply_overrides(load_spec("default"), cost=cost, ranks=n_ranks, steps=steps)
    sc = spec.scenario
    # bench starts at the kick (step 150 of the preset): kick applies at step 0
    return spec, replace(sc, kick=replace(sc.kick, step=0))


def base_particles(spec):
    from paper_2104_11385_b200.workload import kick_velocities, sample_blob

    pos = sample_blob(spec.scenario)
    return pos, kick_velocities(pos, spec.scenario)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        time.sleep(0.15)
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def traffic_per_push():
    """dram read+write bytes per particle from the committed ncu capture."""
    p = ROOT / "profiles" / "ncu_push_kernel.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return float(d["dram_bytes_per_particle"])
    except (KeyError, ValueError):
        return None


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own kernels (oracle/_ref) + oracle port
# ---------------------------------------------------------------------------

def _ref_kernels():
    import importlib.util

    cands = sorted((ROOT / "oracle" / "_ref").glob("_kernels*.so"))
    if cands:
        spec = importlib.util.spec_from_file_location("_kernels", cands[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        return mod, "reference"
    from oracle import lbsim_oracle as O
    return O, "port"


def _cpu_worker(args):
    """One single-threaded reference loop over `reps` replicas of the base
    set (its share of the benchmark workload), whole steps until `seconds`
    elapse.  Returns (pushes, secs, steps)."""
    seconds, cost_kind, reps = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import lbsim_oracle as O
    K, _ = _ref_kernels()
    spec, sc = c2_spec(1, 10 ** 6, "measured")
    pos, vel = base_particles(spec)
    if reps > 1:
        pos = np.ascontiguousarray(np.tile(pos, (reps, 1)))
        vel = np.ascontiguousarray(np.tile(vel, (reps, 1)))
    m = float(sc.box_size)
    nbz = nbx = sc.domain_extent[0] // sc.box_size
    cells = np.full(nbz * nbx, sc.box_size ** 2, dtype=np.int64)
    owner = O.slab_mapping(nbz * nbx, 8)
    pushes, step = 0, 0
    t0 = time.perf_counter()
    while True:
        n = pos.shape[0]
        pos, vel = K.advance_particles(pos, vel, float(sc.domain_extent[0]),
                                       float(sc.domain_extent[1]))
        counts = K.bin_particles(pos, m, nbz, nbx)
        work = O.true_work(counts, sc.box_size, sc.work_weights)
        if cost_kind == "heuristic":
            cost = O.heuristic_cost(counts, cells, 0.75, 0.25)
        else:
            cost = O.measured_cost(work, 0.05, sc.seed, step)
        e, _ = O.efficiency_flagged(cost, owner, 8)
        if step % 10 == 0:
            prop = O.knapsack_assign(cost, 8)
            if O.gate(e, O.efficiency_flagged(cost, prop, 8)[0], 0.10, "relative"):
                owner = prop
        pushes += n
        step += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            return pushes, el, step


def cpu_baseline(seconds: float, processes: int, replicas: int):
    """The reference's CPU path on the benchmark workload: the R replicas of
    the C2 set are split over `processes` single-threaded processes (the
    reference itself is single-threaded), each running whole steps of its
    share for ~`seconds`; value = sum of per-process particle-pushes/s."""
    import multiprocessing as mp

    _, kind = _ref_kernels()
    processes = max(1, min(processes, replicas))
    reps = max(1, replicas // processes)
    if processes <= 1:
        res = [_cpu_worker((seconds, "measured", reps))]
    else:
        with mp.get_context("spawn").Pool(processes) as pool:
            res = pool.map(_cpu_worker, [(seconds, "measured", reps)] * processes)
    value = sum(p / s for p, s, _ in res)
    steps = sum(k for _, _, k in res)
    return {"value": value, "unit": UNIT, "cores": processes, "kind": kind,
            "sample": (f"C2 set (801,499 particles, from the kick) x {reps} replicas per "
                       f"process x {processes} single-threaded processes = "
                       f"{801499 * reps * processes} particles; {steps} whole steps in "
                       f"~{seconds:.0f} s: reference Cython advance_particles + "
                       "bin_particles (oracle/_ref) + measured_cost / efficiency / "
                       "knapsack every 10 (oracle numpy port)")}


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------

def run_reference(args, rank):
    if rank != 0:
        return
    procs = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    cb = cpu_baseline(args.cpu_seconds, procs or 1, args.replicas)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "impl": "reference",
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C2 default.yaml geometry from the kick, x"
                                   f"{args.replicas} replicas (sampled: see cpu_baseline)",
                       "cost": "measured (reference timer model)", "parallelism": "cpu"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_lbx(args, rank, world, local_rank):
    import torch

    from paper_2104_11385_b200 import _lib
    from paper_2104_11385_b200 import device as D
    from paper_2104_11385_b200.workload import Simulation

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1 or args.force_dist:
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29571")
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
        return run_lbx_dist(args, rank, world, dev)
    total = args.warmup + args.steps
    spec, sc = c2_spec(world, total, args.cost)
    pos0, kick0 = base_particles(spec)
    R = args.replicas
    pos = torch.from_numpy(pos0).to(dev).repeat(R, 1)
    kick = torch.from_numpy(kick0).to(dev).repeat(R, 1)
    sim = Simulation(sc, spec.policy, spec.build_provider(), device=dev, positions=pos,
                     kick=kick, time_kernels=True)
    del pos, kick
    n0 = sim.n_init
    sim.run(0, args.warmup)
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    barrier()
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record(stream)
        sim.run(args.warmup, total)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    ms = e0.elapsed_time(e1)
    n_alive = sim.out["n_alive"]
    n_before = np.concatenate(([n0], n_alive[:-1]))
    pushed = float(n_before[args.warmup:total].sum())
    kms = sim.out["kernel_ms"][args.warmup:total]
    res = sim.result()
    if world > 1:
        t = torch.tensor([ms, pushed], dtype=torch.float64, device=dev)
        allt = [torch.zeros_like(t) for _ in range(world)]
        torch.distributed.all_gather(allt, t)
        ms = max(float(x[0]) for x in allt)
        pushed = sum(float(x[1]) for x in allt)
    value = pushed / (ms / 1e3)
    kernel_s = float(np.mean(kms)) / 1e3
    per_launch = float(np.mean(n_before[args.warmup:total]))
    achieved = BYTES_PER_PUSH * per_launch / kernel_s / 1e9
    peak, peak_src = peaks()
    tpp = traffic_per_push()
    effs = [m.efficiency_after for m in res.metrics]

    # ---- the reference's own C2 size (801,499 particles, 1 replica) ----
    c2n = c2_native(args, dev, spec, sc, pos0, kick0)
    c1 = c1_uniform(dev) if not args.no_cpu_baseline else None

    # ---- e2e through the reference-facing C-ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e = e2e_plugin(args, dev, pos0, kick0, R, sc)

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": (f"C2: default.yaml geometry (960x960 cells, 32-cell boxes, "
                                f"900 boxes, blob core 64 / skirt 4 / 55 ppc, seed 7) from "
                                f"the kick, particle set x{R} replicas = {n0} particles per "
                                "GPU"),
                   "cost": spec.build_provider().kind, "lb": "knapsack every 10, 10% rel",
                   "ranks": world, "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                   "l2": "inputs larger than L2 (3.3 GB particle state vs 126 MB L2)"},
        "gpu_launches": 2 * int(args.steps),   # stream_kernel + compaction (exits at once
                                                 # when nothing was absorbed) per step
        "lb": {"ranks": world, "e_first": effs[0] if effs else None,
               "e_mean": float(np.mean(effs)) if effs else None,
               "adoptions": res.summary["adoption_count"]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_src,
                     "kernel": "lbx stream_kernel<clock,pow2,exch=0,push=1>",
                     "bytes_per_launch": BYTES_PER_PUSH * per_launch,
                     "kernel_ms": kernel_s * 1e3,
                     "traffic": None if tpp is None else tpp * per_launch},
        "clocks": clocks.summary(),
        "c2_native": c2n,
        "c1_uniform": c1,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds, 1, args.replicas)
    print(json.dumps(line), flush=True)
    _lib.lib.lbx_sim_destroy(sim.handle)
    sim.handle = None
    del D


def c2_native(args, dev, spec, sc, pos0, kick0, steps=400):
    """The C2 workload at the reference's own size (one replica): a
    latency-bound regime (38 MB of state, L2-resident); whole native loop
    timed with CUDA events."""
    from dataclasses import replace as _replace

    import torch

    from paper_2104_11385_b200.workload import Simulation

    sc1 = _replace(sc, total_steps=steps + 20)
    sim = Simulation(sc1, spec.policy, spec.build_provider(), device=dev,
                     positions=torch.from_numpy(pos0).to(dev), kick=torch.from_numpy(kick0).to(dev))
    sim.run(0, 20)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    sim.run(20, steps + 20)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    n = pos0.shape[0]
    sim.close()
    return {"particles": n, "steps": steps, "us_per_step": 1e3 * ms / steps,
            "pushes_per_s": n * steps / (ms / 1e3),
            "note": "L2-resident, launch/latency bound; incl. host LB loop"}


C1_DOC = dict(scenario_id="c1-uniform", domain=dict(extent=[128, 128], box_size=32), ranks=8,
              blob=dict(center=[64.0, 64.0], core_radius=91.0, edge_scale=0.0,
                        particles_per_cell=8.0),
              kick=dict(step=0, speed=0.0), steps=220, seed=1,
              balance=dict(strategy="knapsack", interval=10, threshold=0.10))


def c1_uniform(dev, steps=200, warm=20):
    """Config C1: 128x128 uniform plasma, 16 boxes, 8 ppc,
    Heuristic + knapsack, 8 ranks -- the case the CPU reference runs; GPU
    native loop vs the reference's compiled kernels + cost/knapsack code on
    one host core, same steps."""
    import time as _t

    import torch

    from oracle import lbsim_oracle as O
    from paper_2104_11385_b200.scenarios import spec_from_dict
    from paper_2104_11385_b200.workload import Simulation

    spec = spec_from_dict(C1_DOC)
    sim = Simulation(spec.scenario, spec.policy, spec.build_provider(), device=dev)
    n = sim.n_init
    sim.run(0, warm)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    sim.run(warm, warm + steps)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    gpu_ms = e0.elapsed_time(e1)
    res = sim.result()
    sim.close()
    K, kind = _ref_kernels()
    cfg = O.config_from_doc(C1_DOC)
    pos, _ = O.init_scenario(cfg["extent"], 32, cfg["center"], 91.0, 0.0, 8.0, 1)
    vel = np.zeros_like(pos)
    owner = O.slab_mapping(16, 8)
    cells = np.full(16, 1024, dtype=np.int64)
    t0 = _t.perf_counter()
    for s in range(steps):
        pos, vel = K.advance_particles(pos, vel, 128.0, 128.0)
        counts = K.bin_particles(pos, 32.0, 4, 4)
        cost = O.heuristic_cost(counts, cells, 0.75, 0.25)
        e, _ = O.efficiency_flagged(cost, owner, 8)
        if s % 10 == 0:
            prop = O.knapsack_assign(cost, 8)
            if O.gate(e, O.efficiency_flagged(cost, prop, 8)[0], 0.10, "relative"):
                owner = prop
    cpu_s = _t.perf_counter() - t0
    return {"particles": n, "steps": steps, "gpu_us_per_step": 1e3 * gpu_ms / steps,
            "gpu_pushes_per_s": n * steps / (gpu_ms / 1e3),
            "cpu_pushes_per_s": n * steps / cpu_s, "cpu_kind": kind, "cpu_cores": 1,
            "mean_efficiency": res.summary["mean_efficiency"],
            "adoptions": res.summary["adoption_count"],
            "note": "L2-resident, latency bound; parity of this config: tests/test_gpu_runs.py::c1"}


def run_lbx_dist(args, rank, world, dev):
    """N > 1: box ownership -> GPU (parallel.DistributedSimulation over NCCL).
    Weak scaling: the C2 set tiled R times per GPU (R*N copies in total),
    initial knapsack mapping, GpuClock costs all-reduced every step, knapsack
    remap every 10 steps with real particle migration on adoption, per-step
    box-crossing exchange."""
    from dataclasses import replace

    import torch
    import torch.distributed as dist

    from paper_2104_11385_b200.parallel import DistributedSimulation, TorchComm

    total = args.warmup + args.steps
    spec, sc = c2_spec(world, total, args.cost)
    sc = replace(sc, initial_mapping="knapsack")
    pos0, kick0 = base_particles(spec)
    R = args.replicas * world
    n_total = pos0.shape[0] * R
    sim = DistributedSimulation(sc, spec.policy, spec.build_provider(), comm=TorchComm(),
                                positions=pos0, kick=kick0, device=dev, replicas=R,
                                capacity=int(1.5 * n_total / world) + 4096)
    sim.run(0, args.warmup)
    stream = torch.cuda.current_stream(dev)
    dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = sim.engine.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clocks:
        e0.record(stream)
        sim.run(args.warmup, total)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = sim.engine.launches - l0
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    res = sim.result()
    n_alive = res.n_alive
    n_before = np.concatenate(([sim.n_init], n_alive[:-1]))
    pushed = float(n_before[args.warmup:total].sum())
    value = pushed / (ms / 1e3)
    effs = [m.efficiency_after for m in res.metrics]
    moved = int(sim.moved[args.warmup:total].sum())
    peak, peak_src = peaks()
    per_gpu_bytes = BYTES_PER_PUSH * pushed / world
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": (f"C2: default.yaml geometry from the kick, particle set x"
                                    f"{R} replicas = {n_total} particles, boxes owned by GPUs"),
                       "cost": spec.build_provider().kind,
                       "lb": "knapsack every 10, 10% rel, initial knapsack",
                       "ranks": world, "parallelism": f"box ownership over {world} GPUs "
                       f"(exchange: {sim.exchange}; p2p = emigrants written into the owner's "
                       f"buffer by the push kernel over NVLink peer memory, NCCL all-reduce)",
                       "l2": "inputs larger than L2"},
            "gpu_launches": int(launches),
            "lb": {"ranks": world, "e_first": effs[0] if effs else None,
                   "e_mean_timed": float(np.mean(effs[args.warmup:])) if effs else None,
                   "adoptions": res.summary["adoption_count"],
                   "particles_migrated_timed": moved},
            "roofline": {"bound": "hbm", "achieved": per_gpu_bytes / (ms / 1e3) / 1e9,
                         "peak": peak, "unit": "GB/s",
                         "frac": per_gpu_bytes / (ms / 1e3) / 1e9 / peak, "peak_source": peak_src,
                         "note": "whole step per GPU (kernels + exchange + host LB)",
                         "traffic": None},
            "clocks": clocks.summary(),
        }
    sim.close()
    del sim
    torch.cuda.empty_cache()
    if not args.no_e2e:
        # e2e at N GPUs: every rank drives the host-buffer plugin path on its
        # own C2 x R set (weak scaling, its own PCIe link), started together;
        # value = all ranks' pushes / the slowest rank's wall time
        dist.barrier()
        e = e2e_plugin(args, dev, pos0, kick0, args.replicas, sc)
        agg = torch.tensor([e["pushed"], e["seconds"], e["h2d_bytes_per_step"],
                            e["d2h_bytes_per_step"]], dtype=torch.float64, device=dev)
        mx = agg.clone()
        dist.all_reduce(agg)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        if rank == 0:
            line["e2e"] = {"value": float(agg[0].item() / mx[1].item()), "unit": UNIT,
                           "h2d_bytes_per_step": int(agg[2].item()),
                           "d2h_bytes_per_step": int(agg[3].item()),
                           "steps": e["steps"], "per_rank": {k: e[k] for k in ("path", "pcie")},
                           "note": "all ranks' host-buffer plugin calls, max wall time over ranks"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def pcie_ceiling(dev, nbytes=1 << 30, reps=3):
    """Measured pinned-host <-> HBM copy rates (GB/s): each direction alone
    and both at once on two streams -- the ceiling of the host-buffer path."""
    import torch
    h = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    d = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2)]
    s = [torch.cuda.Stream(dev) for _ in range(2)]

    def timed(fn):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize(dev)
            best = min(best, time.perf_counter() - t0)
        return best

    def h2d():
        with torch.cuda.stream(s[0]):
            d[0].copy_(h[0], non_blocking=True)

    def d2h():
        with torch.cuda.stream(s[1]):
            h[1].copy_(d[1], non_blocking=True)

    def both():
        h2d()
        d2h()

    t_h, t_d, t_b = timed(h2d), timed(d2h), timed(both)
    return {"h2d_gbs": nbytes / t_h / 1e9, "d2h_gbs": nbytes / t_d / 1e9,
            "bidir_h2d_gbs": nbytes / t_b / 1e9, "bidir_d2h_gbs": nbytes / t_b / 1e9}


def e2e_plugin(args, dev, pos0, kick0, R, sc):
    """Same workload through the reference-facing plugin boundary with HOST
    buffers: every step calls lbx_advance_bin_host (the C-ABI behind
    kernels.advance_particles / bin_particles for host arrays) on the
    particles in pinned host memory -- host->device copy of all particles,
    push + absorb + compaction + per-box counts + heuristic cost, and the
    survivors, counts and costs copied back -- chunked over three streams so
    both PCIe directions overlap the kernels."""
    import torch

    from paper_2104_11385_b200.kernels import advance_bin_host

    n = pos0.shape[0] * R
    nbz = nbx = sc.domain_extent[0] // sc.box_size
    bufs = [torch.empty((n, 2), dtype=torch.float64, pin_memory=True).numpy() for _ in range(4)]
    bufs[0][:] = np.tile(pos0, (R, 1))
    bufs[1][:] = np.tile(kick0, (R, 1))
    state = {"n": n, "inp": (bufs[0], bufs[1]), "out": (bufs[2], bufs[3])}
    ez, ex = float(sc.domain_extent[0]), float(sc.domain_extent[1])
    io = {"h2d": 0, "d2h": 0}

    def step():
        k = state["n"]
        ip, iv = state["inp"]
        op, ov = state["out"]
        p, v, counts, cost = advance_bin_host(ip[:k], iv[:k], ez, ex, float(sc.box_size),
                                              nbz, nbx, out=(op, ov), dev=dev)
        m = p.shape[0]
        io["h2d"] += 32 * k
        io["d2h"] += 32 * m + 16 * nbz * nbx
        state["n"] = m
        state["inp"], state["out"] = state["out"], state["inp"]
        return k

    for _ in range(2):
        step()
    io["h2d"] = io["d2h"] = 0
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    pushed = sum(step() for _ in range(args.e2e_steps))
    el = time.perf_counter() - t0
    ceil = pcie_ceiling(dev)
    h2d, d2h = io["h2d"] / args.e2e_steps, io["d2h"] / args.e2e_steps
    # the e2e roofline: both directions at the measured concurrent copy rates
    t_min = max(h2d / (ceil["bidir_h2d_gbs"] * 1e9), d2h / (ceil["bidir_d2h_gbs"] * 1e9))
    bound = (pushed / args.e2e_steps) / t_min
    return {"value": pushed / el, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "steps": args.e2e_steps, "seconds": el, "pushed": pushed,
            "pcie": dict(ceil, bound_pushes_per_s=bound, frac_of_bound=(pushed / el) / bound),
            "path": "lbx_advance_bin_host (reference AoS layout, pinned host buffers, "
                    "4 Mi-particle chunks over 3 streams, no host round trip per chunk), copies in the timed region"}


def main():
    # one JSON line on stdout: keep NCCL's version banner off it unless the
    # user asked for NCCL debugging
    if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
        os.environ["NCCL_DEBUG"] = "WARN"
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    run_lbx(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
