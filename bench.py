#!/usr/bin/env python
"""Benchmark: particle-pushes/s including in-situ cost assessment, plus LB
efficiency, on B200 (BASELINE.json metric; workload = config C2).

Workload (config C2, "2D laser-ion dense-slab target, GpuClock costs,
dynamic LB every 10 steps"): the reference's default.yaml geometry -- 960x960
cells, 32-cell boxes (900 boxes), dense blob (core 64, skirt 4, 55 ppc)
sampled with the reference's own PCG64 stream -- from the kick step onward
(radial kick, speed 0.035, drift 0.01), 8 virtual ranks (N > 1: one rank per
GPU), initial slab mapping, knapsack remap attempted every 10 steps with a
10 % relative threshold.  To fill a B200 the 801,499-particle set is tiled R
times (default R=128 -> 102.6 M particles, 3.3 GB of particle state): every
replica evolves identically, so per-box counts are exactly R x the
reference's (tests/test_gpu_bench_parity).

Both arms print the SAME `config` dict (bench_config):
* B200 arm: the fused sm_100a kernel (push + absorb + stable compaction +
  per-box counts + heuristic cost + GpuClock clock64 tally) + the step record
  written to mapped host memory + the native host loop (cost vector,
  efficiency over the 8 ranks, knapsack attempt every 10 steps).  Inputs
  (3.3 GB) are larger than L2 (126 MB), so no flush is needed between steps.
* `e2e`: the same steps through the reference-facing plugin (C-ABI
  lbx_advance_bin_host with pinned HOST buffers: H2D of every particle, D2H
  of the survivors + counts every step) driving the package's public
  balancer API (true_work -> measured_cost -> efficiency -> knapsack every
  10), i.e. the reference's run loop with its kernels swapped.
* --impl reference: the reference's own compiled Cython kernels
  (oracle/_ref) + the oracle port of its numpy cost / balancer code, with
  GpuClock costs modelled the way the reference models them (measured_cost,
  cost.py:98-113) -- the package is NOT imported on this arm; one process per
  host core, each on a bounded sample of the workload; rank 0 only.

--gpus N without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (NCCL INIT logging on).
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
    ap.add_argument("--ranks", type=int, default=8,
                    help="virtual ranks of the distribution mapping at N=1 (N>1: one per GPU)")
    ap.add_argument("--e2e-steps", type=int, default=None, help="default: --steps")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pic", action="store_true", help="skip the PIC (north-star item 1) line")
    ap.add_argument("--no-native", action="store_true",
                    help="skip the native-size lines (resident multi-step kernel): "
                         "profiling runs (ncu serialises the kernel's host handshake)")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the multi-GPU box-ownership path even at N=1 (testing)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# workload (shared by both arms; nothing here imports the package)
# ---------------------------------------------------------------------------

BASE_PARTICLES = 801_499   # the C2 set (default.yaml blob), tests/golden


def c2_doc(provider: str, ranks: int, steps: int, initial_mapping: str = "slab") -> dict:
    """default.yaml (reference pkg/src/lbsim/scenarios/default.yaml) with the
    kick moved to step 0 (the bench starts at the kick), `ranks` virtual ranks
    and the cost provider of the arm."""
    return dict(scenario_id="c2-bench", domain=dict(extent=[960, 960], box_size=32),
                ranks=int(ranks),
                blob=dict(center=[480.0, 480.0], core_radius=64.0, edge_scale=4.0,
                          particles_per_cell=55.0),
                kick=dict(step=0, speed=0.035, drift=0.01), steps=int(steps),
                compute_fraction=0.5, work_weights=[0.75, 0.25],
                initial_mapping=initial_mapping, seed=7,
                balance=dict(strategy="knapsack", interval=10, threshold=0.10,
                             threshold_mode="relative", cap_factor=1.5),
                provider=dict(kind=provider, weights="default", noise=0.05,
                              instrumented_overhead=2.0))


def dist_mode(args, world: int) -> bool:
    return world > 1 or args.force_dist


def bench_ranks(args, world: int) -> int:
    return world if dist_mode(args, world) else args.ranks


def bench_initial_mapping(args, world: int) -> str:
    # N > 1: the ranks are real GPUs; a knapsack start keeps the first steps
    # from piling the blob onto two GPUs (both arms use the same rule)
    return "knapsack" if dist_mode(args, world) else "slab"


def bench_config(args, world: int) -> dict:
    """The `config` dict printed by BOTH arms (same workload, same mapping)."""
    R = args.replicas
    return {"workload": (f"C2: default.yaml geometry (960x960 cells, 32-cell boxes, 900 boxes, "
                         f"blob core 64 / skirt 4 / 55 ppc, seed 7) from the kick, particle "
                         f"set x{R} replicas = {BASE_PARTICLES * R} particles per GPU"),
            "ranks": bench_ranks(args, world),
            "cost": ("GpuClock: clock64 tally fused in the B200 push kernel; the CPU "
                     "reference arm uses the reference's model of it (measured_cost, "
                     "cost.py:98-113, noise 0.05)"),
            "lb": (f"knapsack (cap 1.5) every 10 steps, 10% relative threshold, initial "
                   f"{bench_initial_mapping(args, world)} mapping"),
            "steps": args.steps, "warmup": args.warmup,
            "l2": "inputs larger than L2 (3.3 GB particle state per GPU vs 126 MB L2)"}


def c2_spec(n_ranks: int, steps: int, cost: str, initial_mapping: str = "slab"):
    """Package RunSpec + ScenarioConfig of the C2 bench workload."""
    from paper_2104_11385_b200.scenarios import spec_from_dict

    spec = spec_from_dict(c2_doc(cost, n_ranks, steps, initial_mapping))
    return spec, spec.scenario


def arm_spec(args, world: int, steps: int):
    """The B200 arm's spec (the config bench_config describes)."""
    return c2_spec(bench_ranks(args, world), steps, args.cost,
                   bench_initial_mapping(args, world))


def base_particles(spec):
    from paper_2104_11385_b200.workload import kick_velocities, sample_blob

    pos = sample_blob(spec.scenario)
    return pos, kick_velocities(pos, spec.scenario)


def oracle_particles(cfg):
    """The same C2 set from the oracle (reference arm: no package import)."""
    from oracle import lbsim_oracle as O

    pos, _ = O.init_scenario(cfg["extent"], cfg["box_size"], cfg["center"],
                             cfg["core_radius"], cfg["edge_scale"], cfg["ppc"], cfg["seed"])
    vel = O.kick_velocities(pos, cfg["center"], cfg["kick_speed"], cfg["kick_drift"],
                            cfg["seed"])
    return pos, vel


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


def _cpu_worker(a):
    """One single-threaded reference loop over `reps` replicas of the base set
    (its sample of the benchmark workload), whole steps until `seconds`
    elapse.  The workload is R identical replicas, so the full workload's
    per-box counts are exactly (R / reps) x the sample's: the cost, efficiency
    and knapsack steps run on that full vector, i.e. the same LB decisions as
    the B200 arm's.  Returns (pushes, secs, steps, lb dict)."""
    seconds, reps, R, ranks, init_map = a
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import lbsim_oracle as O
    K, _ = _ref_kernels()
    cfg = O.config_from_doc(c2_doc("measured", ranks, 10 ** 6, init_map))
    pos, vel = oracle_particles(cfg)
    if reps > 1:
        pos = np.ascontiguousarray(np.tile(pos, (reps, 1)))
        vel = np.ascontiguousarray(np.tile(vel, (reps, 1)))
    scale = max(1, R // reps)
    m, wts = cfg["box_size"], cfg["work_weights"]
    ez, ex = (float(v) for v in cfg["extent"])
    nbz, nbx = cfg["extent"][0] // m, cfg["extent"][1] // m
    counts0 = K.bin_particles(pos, float(m), nbz, nbx) * scale
    if init_map == "slab":
        owner = O.slab_mapping(nbz * nbx, ranks)
    else:
        owner = O.knapsack_assign(O.true_work(counts0, m, wts), ranks)
    pushes, step, effs, adoptions = 0, 0, [], 0
    t0 = time.perf_counter()
    while True:
        n = pos.shape[0]
        pos, vel = K.advance_particles(pos, vel, ez, ex)
        counts = K.bin_particles(pos, float(m), nbz, nbx) * scale
        work = O.true_work(counts, m, wts)
        cost = O.measured_cost(work, cfg["noise"], cfg["seed"], step)
        e, _ = O.efficiency_flagged(cost, owner, ranks)
        if step % cfg["interval"] == 0:
            prop = O.knapsack_assign(cost, ranks, cfg["cap_factor"])
            ep = O.efficiency_flagged(cost, prop, ranks)[0]
            if O.gate(e, ep, cfg["threshold"], cfg["threshold_mode"]):
                owner, e = prop, ep
                adoptions += 1
        effs.append(e)
        pushes += n
        step += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            return pushes, el, step, {"e_first": effs[0], "e_mean": float(np.mean(effs)),
                                      "adoptions": adoptions, "steps": step}


def cpu_baseline(seconds: float, processes: int, args, world: int):
    """The reference's CPU path on the benchmark workload: the R replicas of
    the C2 set are split over `processes` single-threaded processes (the
    reference itself is single-threaded), each running whole steps of its
    share for ~`seconds`; value = sum of per-process particle-pushes/s."""
    import multiprocessing as mp

    _, kind = _ref_kernels()
    R = args.replicas * (world if dist_mode(args, world) else 1)   # whole job
    processes = max(1, min(processes, R))
    reps = max(1, R // processes)
    job = (seconds, reps, R, bench_ranks(args, world), bench_initial_mapping(args, world))
    if processes <= 1:
        res = [_cpu_worker(job)]
    else:
        with mp.get_context("spawn").Pool(processes) as pool:
            res = pool.map(_cpu_worker, [job] * processes)
    value = sum(r[0] / r[1] for r in res)
    steps = sum(r[2] for r in res)
    return {"value": value, "unit": UNIT, "cores": processes, "kind": kind,
            "sample": (f"C2 set ({BASE_PARTICLES:,} particles, from the kick) x {reps} "
                       f"replicas per process x {processes} single-threaded processes = "
                       f"{BASE_PARTICLES * reps * processes} particles; {steps} whole steps in "
                       f"~{seconds:.0f} s: reference Cython advance_particles + "
                       "bin_particles (oracle/_ref) + true_work / measured_cost / "
                       "efficiency / knapsack every 10 on the full workload's per-box "
                       "counts (oracle numpy port)"),
            "lb": res[0][3]}


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------

def run_reference(args, rank, world):
    """The reference arm: never imports paper_2104_11385_b200 (no libLBX)."""
    if rank != 0:
        return
    procs = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    cb = cpu_baseline(args.cpu_seconds, procs or 1, args, world)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "impl": "reference",
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": bench_config(args, world),
            "lb": cb.pop("lb"),
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
    spec, sc = arm_spec(args, world, total)
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
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record(stream)
        sim.run(args.warmup, total)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    n_alive = sim.out["n_alive"]
    n_before = np.concatenate(([n0], n_alive[:-1]))
    pushed = float(n_before[args.warmup:total].sum())
    kms = sim.out["kernel_ms"][args.warmup:total]
    res = sim.result()
    value = pushed / (ms / 1e3)
    kernel_s = float(np.mean(kms)) / 1e3
    per_launch = float(np.mean(n_before[args.warmup:total]))
    achieved = BYTES_PER_PUSH * per_launch / kernel_s / 1e9
    peak, peak_src = peaks()
    tpp = traffic_per_push()
    effs = [m.efficiency_after for m in res.metrics]
    adopt_timed = int(sum(m.adopted for m in res.metrics[args.warmup:total]))
    sim.close()
    del sim
    torch.cuda.empty_cache()

    # ---- the reference's own C2 size (801,499 particles, 1 replica) ----
    c2n = c2_native(args, dev, spec, sc, pos0, kick0) if not args.no_native else None
    c1 = c1_uniform(dev) if not (args.no_cpu_baseline or args.no_native) else None
    comp = compaction_leavers(dev) if not args.no_e2e else None
    picl = None
    if not args.no_pic:
        try:   # an extra line: never let it take the headline line down
            picl = pic_line(dev, pos0, kick0, R, sc)
        except Exception as e:   # noqa: BLE001
            picl = {"error": f"{type(e).__name__}: {e}"}
            torch.cuda.empty_cache()

    # ---- e2e through the reference-facing C-ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e = e2e_plugin(args, dev, pos0, kick0, R, spec)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(args, world),
        "parallelism": "1 GPU, 8 virtual ranks (distribution mapping only)",
        "gpu_launches": 2 * int(args.steps),   # stream_kernel + compaction (exits at once
                                                 # when nothing was absorbed) per step
        "lb": {"ranks": sc.n_ranks, "e_first": effs[0] if effs else None,
               "e_mean": float(np.mean(effs)) if effs else None,
               "e_mean_timed": float(np.mean(effs[args.warmup:total])) if effs else None,
               "adoptions": res.summary["adoption_count"], "adoptions_timed": adopt_timed},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_src,
                     "kernel": "lbx stream_kernel<clock,pow2,exch=0,push=1>",
                     "bytes_per_launch": BYTES_PER_PUSH * per_launch,
                     "kernel_ms": kernel_s * 1e3,
                     "traffic": None if tpp is None else tpp * per_launch},
        "clocks": clocks.summary(),
        "c2_native": c2n,
        "c1_uniform": c1,
        "compaction": comp,
        "pic": picl,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds, 1, args, world)
        line["cpu_baseline"].pop("lb", None)
    print(json.dumps(line), flush=True)
    del D, _lib


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
    resident = sim.resident_runs
    sim.close()
    return {"particles": n, "steps": steps, "us_per_step": 1e3 * ms / steps,
            "pushes_per_s": n * steps / (ms / 1e3),
            "resident_runs": resident,
            "note": "resident kernel (particles in shared memory across steps, lbx_resident.cu); "
                    "incl. the host LB loop (8-rank GpuClock knapsack every 10)"}


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
    resident = sim.resident_runs
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
            "resident_runs": resident,
            "note": "resident kernel (lbx_resident.cu); parity of this config: "
                    "tests/test_gpu_runs.py::c1, tests/test_gpu_resident.py"}


def pic_line(dev, pos0, kick0, R, sc, steps=10, warmup=3, resort=10):
    """North-star item 1 (SURVEY 8d "PIC extension"): the same C2 particle set
    (x R) through the 2D3V PIC push + deposit, tolerance mode (pic_pipe_kernel,
    the fields of a 960^2 Yee grid; bench_pic.py has every mode).  `steps`
    steps run back to back (no host round trip) with a cell sort every
    `resort` steps, the sorts inside the timed region; the first step after
    a sort is also timed alone.  80 B per push (5 fp64 read + write)."""
    import torch

    from paper_2104_11385_b200 import device, pic

    dt = 0.5
    n = pos0.shape[0] * R
    u0 = np.column_stack([kick0[:, 0] / dt, kick0[:, 1] / dt, np.zeros(len(kick0))])
    nz, nx = sc.domain_extent
    st = pic.PicState.create(pos0[:1], u0[:1], nz, nx, device=dev)
    cols = (pos0[:, 0], pos0[:, 1], u0[:, 0], u0[:, 1], u0[:, 2])
    for name, col in zip(("z", "x", "uz", "ux", "uy"), cols):
        t = torch.zeros(n + 2, dtype=torch.float64, device=dev)
        t[:n].copy_(torch.from_numpy(np.ascontiguousarray(col)).to(dev).repeat(R))
        setattr(st, name, t)
    st.n = n
    ctx = device.Context(dev, capacity=n)
    kw = dict(clock=True, field_solve=False, fast=True, sync=False)
    stream = torch.cuda.current_stream(dev)
    pic.pic_sort(ctx, st)
    for _ in range(warmup):
        pic.pic_step(ctx, st, sc.box_size, -1.0, -1e-4, dt, **kw)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(stream)
    for i in range(steps):
        if i % resort == 0:
            pic.pic_sort(ctx, st, sync=False)   # inside the timed region
        if i == 0:
            e[1].record(stream)
        pic.pic_step(ctx, st, sc.box_size, -1.0, -1e-4, dt, **kw)
        if i == 0:
            e[2].record(stream)
    e[3].record(stream)
    torch.cuda.synchronize(dev)
    n1 = pic.pic_sync(ctx, st)
    peak, _ = peaks()
    first_ms = e[1].elapsed_time(e[2])   # the first step after the sort
    ms = e[0].elapsed_time(e[3]) / steps
    del st, ctx
    torch.cuda.empty_cache()
    return {"workload": f"C2 set x{R} = {n} particles, 2D3V PIC push + deposit, {nz}x{nx} "
                        "Yee grid, tolerance mode (LBX_PIC_FAST), GpuClock on",
            "bytes_per_particle": 80, "steps": steps, "resort_every": resort,
            "ms_per_step": ms, "pushes_per_s": n / (ms / 1e3),
            "frac_of_hbm": 80.0 * n / (ms / 1e3) / 1e9 / peak,
            "first_step_after_sort_ms": first_ms,
            "first_step_frac_of_hbm": 80.0 * n / (first_ms / 1e3) / 1e9 / peak,
            "survivors": n1, "kernel": "pic_pipe_kernel<clock, fast> (+ quad copy, current "
                                      "gather, hole filling per step; cell sort every "
                                      f"{resort} steps)"}


def compaction_leavers(dev, n=100_000_000, steps=3, ext=960.0, box=32.0):
    """Leaver-heavy steps: n particles uniform over the
    C2 domain, v ~ N(0, 2 cells/step), in random order, so ~0.7 % are
    absorbed every step from anywhere in the array and the stable look-back
    compaction (scan_kernel<COMPACT_SOA>) re-packs essentially all of it:
    64 B per particle at or after the first absorbed index (read + write
    z, x, vz, vx).  Compaction time = step time (events) - fused kernel time
    (lbx_ctx_last_kernel_ms)."""
    import ctypes as C

    import torch

    from paper_2104_11385_b200 import _lib
    from paper_2104_11385_b200 import device as D

    g = torch.Generator(device=dev).manual_seed(7)
    st = D.ParticleState.empty(n, dev)
    for t in (st.z, st.x):
        t[:n].copy_(torch.rand(n, generator=g, device=dev, dtype=torch.float64) * ext)
    for t in (st.vz, st.vx):
        t[:n].copy_(torch.randn(n, generator=g, device=dev, dtype=torch.float64) * 2.0)
    st.n = n
    ctx = D.Context(dev, capacity=n)
    _lib.check(_lib.lib.lbx_ctx_enable_timing(ctx.handle, 1))
    nbz = nbx = int(ext // box)
    D.push_step(ctx, st, ext, ext, box, nbz, nbx)       # warm-up (allocations)
    rows = []
    stream = torch.cuda.current_stream(dev)
    for _ in range(steps):
        n0 = st.n
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        D.push_step(ctx, st, ext, ext, box, nbz, nbx)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        km = C.c_float()
        _lib.check(_lib.lib.lbx_ctx_last_kernel_ms(ctx.handle, C.byref(km)))
        step_ms = e0.elapsed_time(e1)
        comp_ms = max(step_ms - km.value, 1e-6)
        rows.append({"n_before": n0, "absorbed": n0 - st.n, "step_ms": step_ms,
                     "push_kernel_ms": km.value, "compaction_ms": comp_ms,
                     "compaction_gbs": 64.0 * n0 / (comp_ms / 1e3) / 1e9})
    peak, _ = peaks()
    gbs = float(np.mean([r["compaction_gbs"] for r in rows]))
    del st, ctx
    torch.cuda.empty_cache()
    return {"workload": f"{n} particles uniform over 960x960, v ~ N(0, 2) cells/step, random "
                        "order (absorbed from anywhere in the array)",
            "bytes_per_particle": 64, "compaction_gbs": gbs, "frac_of_hbm": gbs / peak,
            "steps": rows,
            "kernel": "scan_kernel<COMPACT_SOA> (decoupled look-back stable compaction)"}


def run_lbx_dist(args, rank, world, dev):
    """N > 1: box ownership -> GPU (parallel.DistributedSimulation over NCCL).
    Weak scaling: the C2 set tiled R times per GPU (R*N copies in total),
    initial knapsack mapping, GpuClock costs all-reduced every step, knapsack
    remap every 10 steps with real particle migration on adoption, per-step
    box-crossing exchange."""
    import torch
    import torch.distributed as dist

    from paper_2104_11385_b200.parallel import DistributedSimulation, TorchComm

    total = args.warmup + args.steps
    spec, sc = arm_spec(args, world, total)
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
            "config": bench_config(args, world),
            "parallelism": (f"box ownership over {world} GPUs, {n_total} particles in total "
                            f"(exchange: {sim.exchange}; p2p = emigrants written into the "
                            f"owner's buffer by the push kernel over NVLink peer memory, NCCL "
                            f"all-reduce)"),
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
        e = e2e_plugin(args, dev, pos0, kick0, args.replicas, spec)
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


def e2e_plugin(args, dev, pos0, kick0, R, spec):
    """Same workload through the reference-facing plugin boundary with HOST
    buffers -- the reference's run loop (workload.py:411-439) with its kernel
    backend swapped: every step calls lbx_advance_bin_host (the C-ABI behind
    kernels.advance_particles / bin_particles for host arrays) on the
    particles in pinned host memory -- host->device copy of all particles,
    push + absorb + compaction + per-box counts, survivors and counts copied
    back, chunked over three streams so both PCIe directions overlap the
    kernels -- then the package's public API on the host: true_work ->
    measured_cost (the GpuClock model; no clock on host buffers) ->
    efficiency -> knapsack attempt every 10 steps with the gate."""
    import torch

    from paper_2104_11385_b200.balancer import attempt_rebalance, efficiency
    from paper_2104_11385_b200.cost import MeasurementConfig, measured_cost
    from paper_2104_11385_b200.workload import box_array_for, initial_mapping, true_work

    sc, policy = spec.scenario, spec.policy
    steps = args.e2e_steps or args.steps
    n = pos0.shape[0] * R
    nbz = nbx = sc.domain_extent[0] // sc.box_size
    bufs = [torch.empty((n, 2), dtype=torch.float64, pin_memory=True).numpy() for _ in range(4)]
    bufs[0][:] = np.tile(pos0, (R, 1))
    bufs[1][:] = np.tile(kick0, (R, 1))
    ba = box_array_for(sc)
    from paper_2104_11385_b200.kernels import advance_bin_host, bin_particles
    counts0 = bin_particles(bufs[0], float(sc.box_size), nbz, nbx)
    state = {"n": n, "inp": (bufs[0], bufs[1]), "out": (bufs[2], bufs[3]),
             "dm": initial_mapping(sc, ba, counts0), "step": 0, "adopt": 0, "eff": []}
    mcfg = MeasurementConfig(noise_amplitude=0.05, seed=sc.seed)
    ez, ex = float(sc.domain_extent[0]), float(sc.domain_extent[1])
    io = {"h2d": 0, "d2h": 0}

    def step():
        k = state["n"]
        ip, iv = state["inp"]
        op, ov = state["out"]
        p, v, counts, _ = advance_bin_host(ip[:k], iv[:k], ez, ex, float(sc.box_size),
                                           nbz, nbx, out=(op, ov), dev=dev)
        m = p.shape[0]
        io["h2d"] += 32 * k
        io["d2h"] += 32 * m + 16 * nbz * nbx
        state["n"] = m
        state["inp"], state["out"] = state["out"], state["inp"]
        s = state["step"]
        cv = measured_cost(true_work(counts, sc), mcfg, s)
        out = attempt_rebalance(cv, state["dm"], policy, s)
        if out.adopted:
            state["dm"] = out.proposed
            state["adopt"] += 1
        state["eff"].append(out.efficiency_proposed if out.adopted
                            else out.efficiency_current)
        state["step"] = s + 1
        return k

    for _ in range(2):
        step()
    io["h2d"] = io["d2h"] = 0
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    pushed = sum(step() for _ in range(steps))
    el = time.perf_counter() - t0
    ceil = pcie_ceiling(dev)
    h2d, d2h = io["h2d"] / steps, io["d2h"] / steps
    # the e2e roofline: both directions at the measured concurrent copy rates
    t_min = max(h2d / (ceil["bidir_h2d_gbs"] * 1e9), d2h / (ceil["bidir_d2h_gbs"] * 1e9))
    bound = (pushed / steps) / t_min
    return {"value": pushed / el, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "steps": steps, "seconds": el, "pushed": pushed,
            "lb": {"e_first": state["eff"][0], "adoptions": state["adopt"]},
            "pcie": dict(ceil, bound_pushes_per_s=bound, frac_of_bound=(pushed / el) / bound),
            "path": ("lbx_advance_bin_host (reference AoS layout, pinned host buffers, "
                     "4 Mi-particle chunks over 3 streams) + the package's balancer API "
                     "(true_work, measured_cost, efficiency, knapsack every 10) on the "
                     "host; copies in the timed region")}


def self_launch(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-exec under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible",
              file=sys.stderr, flush=True)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    # NCCL INIT logging on (communicator lines with nranks); the JSON line is
    # printed last, after every NCCL init message
    if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
        os.environ["NCCL_DEBUG"] = "INFO"
    sub = os.environ.get("NCCL_DEBUG_SUBSYS", "")
    if sub and "INIT" not in sub.upper() and sub.upper() != "ALL":
        os.environ["NCCL_DEBUG_SUBSYS"] = sub + ",INIT"
    elif not sub:
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, max(world, args.gpus))
        return
    if "WORLD_SIZE" not in os.environ and (args.gpus > 1 or args.force_dist):
        sys.exit(self_launch(args))
    if world != args.gpus:
        print(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}",
              file=sys.stderr, flush=True)
        sys.exit(2)
    run_lbx(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
