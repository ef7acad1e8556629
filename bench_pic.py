#!/usr/bin/env python
"""PIC push + deposit benchmark (north-star item 1; SURVEY 8d "PIC extension").

Workload: the C2 blob (default.yaml geometry: 960x960 cells, 32-cell boxes,
801,499 particles sampled with the reference's stream) tiled R times
(default 128 -> 102.6 M macro-particles), momenta from the C2 kick velocity
(u = v/dt), electrons (q/m = -1), dt = 0.5, GpuClock tally on.  Every mode
starts from the same initial particles.  Timed with CUDA events on the
launch stream:
  push_deposit          lbx_pic_step, sorted mode (sort-on-write), with
                        LBX_PIC_NO_FIELD_SOLVE: quad fields + gather + Boris +
                        deposit + counts/clock + compaction + cell-slot scan;
  push_deposit_inplace  the same in place (order kept, no sorting: the
                        deposit's cell runs decay as particles drift);
  push_deposit_noclock  sorted mode without the GpuClock tally (its overhead
                        is gpuclock_overhead = push_deposit / this - 1);
  full_step             sorted mode plus the Yee update;
  push_deposit_resort   in place with lbx_pic_sort (cell counting sort)
                        every --resort steps, its cost inside the timed step;
  push_deposit_tiled    the same with the tile-major sort and LBX_PIC_TILED
                        steps (shared-memory patch and current);
  push_deposit_fast     in place, tolerance mode (LBX_PIC_FAST: float32
                        Boris increment, FMA gathers);
  push_deposit_fast_resort  the same with lbx_pic_sort every --resort steps;
  push_deposit_resort_noclock / push_deposit_fast_resort_noclock /
  push_deposit_esk3_resort_noclock
                        the same without the GpuClock tally (overhead =
                        gpuclock_overhead_<mode>, pipelined step times);
  push_deposit_fast_resort_quad  push_deposit_fast_resort with the quad copy
                        forced (the pipelined kernel on a sparse plasma);
  push_deposit_fast_tiled   tolerance mode on the tiled path (tile-major sort
                        every --resort steps; sparse plasmas);
  push_deposit_esk1/esk3  charge-conserving Esirkepov deposition with shape
                        order 1 / 3 (the paper's order) and
                        same-order gather, in place (+ _resort: cell sort
                        every --resort steps; full_step_esk3_resort adds the
                        Yee update).
Roofline: HBM, algorithmic bytes = 80 B per particle (read z,x,uz,ux,uy +
write them, float64) -- field patch and current flush traffic is counted
separately from ncu (profiles/).  Prints one JSON object.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BYTES_PER_PARTICLE = 80


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replicas", type=int, default=128)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=["c2", "uniform"],
                    help="c2: the C2 blob tiled (dense, ~7,000 particles per occupied cell); "
                         "uniform: SURVEY 8d's roofline plasma, 4096x4096 cells x 8 ppc "
                         "(134 M particles), thermal momenta")
    ap.add_argument("--resort", type=int, default=25,
                    help="push_deposit_resort: lbx_pic_sort every this many steps")
    ap.add_argument("--modes", default="push_deposit,push_deposit_inplace,push_deposit_noclock,"
                                        "full_step,push_deposit_resort",
                    help="comma-separated subset of the modes")
    args = ap.parse_args()

    import torch

    import bench
    from paper_2104_11385_b200 import device, pic

    dev = torch.device("cuda:0")
    dt = 0.5
    if args.workload == "c2":
        spec, sc = bench.c2_spec(1, 10, "gpuclock")
        pos0, kick0 = bench.base_particles(spec)
        u0 = np.column_stack([kick0[:, 0] / dt, kick0[:, 1] / dt, np.zeros(len(kick0))])
        R = args.replicas
        nz, nx = sc.domain_extent
        box = sc.box_size
        label = (f"C2 blob x{R} replicas = {pos0.shape[0] * R} particles, 960x960 Yee grid, "
                 f"box 32, dt {dt}, q/m -1, GpuClock on")
    else:   # uniform plasma, cell-sorted, 8 per cell, thermal u ~ N(0, 0.05)
        nz = nx = 4096
        ppc, R, box = 8, 1, 128
        rng = np.random.default_rng(42)
        cell = np.repeat(np.arange(nz * nx, dtype=np.int64), ppc)
        off = rng.random((cell.size, 2))
        pos0 = np.column_stack([(cell // nx) + off[:, 0], (cell % nx) + off[:, 1]])
        u0 = rng.normal(0.0, 0.05, size=(cell.size, 3))
        del cell, off
        label = (f"uniform plasma 4096x4096 cells x {ppc} ppc = {pos0.shape[0]} particles, "
                 f"box {box}, thermal u ~ N(0, 0.05), dt {dt}, q/m -1, GpuClock on")
    n = pos0.shape[0] * R
    cols = (("z", pos0[:, 0]), ("x", pos0[:, 1]), ("uz", u0[:, 0]), ("ux", u0[:, 1]),
            ("uy", u0[:, 2]))
    init = {}
    for name, col in cols:   # tile on the device (host arrays of 100 M particles are not needed)
        t = torch.zeros(n + 2, dtype=torch.float64, device=dev)
        t[:n].copy_(torch.from_numpy(np.ascontiguousarray(col)).to(dev).repeat(R))
        init[name] = t
    ctx = device.Context(dev, capacity=n)
    peak, peak_src = bench.peaks()
    out = {"workload": label, "particles": n}
    stream = torch.cuda.current_stream(dev)
    for mode, solve, sort, clk in (("push_deposit", False, True, True),
                                   ("push_deposit_inplace", False, False, True),
                                   ("push_deposit_noclock", False, True, False),
                                   ("full_step", True, True, True),
                                   ("push_deposit_resort", False, False, True),
                                   ("push_deposit_resort_noclock", False, False, False),
                                   ("push_deposit_tiled", False, False, True),
                                   ("push_deposit_fast", False, False, True),
                                   ("push_deposit_fast_resort", False, False, True),
                                   ("push_deposit_fast_resort_noclock", False, False, False),
                                   ("push_deposit_fast_tiled", False, False, True),
                                   ("push_deposit_fast_resort_quad", False, False, True),
                                   ("push_deposit_esk1", False, False, True),
                                   ("push_deposit_esk3", False, False, True),
                                   ("push_deposit_esk3_resort", False, False, True),
                                   ("push_deposit_esk3_resort_noclock", False, False, False),
                                   ("full_step_esk3_resort", True, False, True)):
        if mode not in args.modes.split(","):
            continue
        st = pic.PicState.create(pos0[:1], u0[:1], nz, nx, device=dev)
        for name, t in init.items():
            setattr(st, name, t.clone())
        st.n = n
        resort = mode in ("push_deposit_resort", "push_deposit_resort_noclock", "push_deposit_tiled", "push_deposit_fast_tiled",
                          "push_deposit_fast_resort", "push_deposit_fast_resort_noclock",
                          "push_deposit_fast_resort_quad",
                          "push_deposit_esk3_resort_noclock") or mode.endswith("esk3_resort")
        order = 3 if "esk3" in mode else (1 if "esk1" in mode else 0)
        tiled = mode in ("push_deposit_tiled", "push_deposit_fast_tiled")
        fast = mode.startswith("push_deposit_fast")
        if resort:   # start cell-ordered, like the other modes' first sorted step
            pic.pic_sort(ctx, st, tiled=tiled)
        for w in range(args.warmup):
            try:
                pic.pic_step(ctx, st, box, -1.0, -1e-4, dt, clock=clk, field_solve=solve,
                             sort=sort, tiled=tiled, fast=fast, shape_order=order,
                             gather="quad" if mode.endswith("_quad") else None)
            except ValueError as e:
                raise ValueError(f"mode {mode} warm-up step {w}: {e}") from None
        times = []
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n_before = st.n
            e0.record(stream)
            if resort and (len(times) + args.warmup) % args.resort == 0:
                pic.pic_sort(ctx, st, tiled=tiled)
            try:
                pic.pic_step(ctx, st, box, -1.0, -1e-4, dt, clock=clk, field_solve=solve,
                             sort=sort, tiled=tiled, fast=fast, shape_order=order,
                             gather="quad" if mode.endswith("_quad") else None)
            except ValueError as e:
                raise ValueError(f"mode {mode} step {len(times)}: {e}") from None
            e1.record(stream)
            torch.cuda.synchronize(dev)
            times.append((e0.elapsed_time(e1), n_before))
        ms = float(np.mean([t for t, _ in times]))
        nb = float(np.mean([k for _, k in times]))
        achieved = BYTES_PER_PARTICLE * nb / (ms / 1e3) / 1e9
        out[mode] = {"ms": ms, "ms_per_step": [round(t, 3) for t, _ in times],
                     "pushes_per_s": nb / (ms / 1e3), "achieved_gbs": achieved,
                     "frac_of_hbm_peak": achieved / peak}
        # the same steps back to back (sync=False: no host readback between
        # steps): the device time of a step, without the per-step host round
        # trip the loop above includes
        del st
        st = pic.PicState.create(pos0[:1], u0[:1], nz, nx, device=dev)
        for name, t in init.items():
            setattr(st, name, t.clone())
        st.n = n
        if resort:
            pic.pic_sort(ctx, st, tiled=tiled)
        gather = "quad" if mode.endswith("_quad") else None
        kw = dict(clock=clk, field_solve=solve, sort=sort, tiled=tiled, fast=fast,
                  shape_order=order, gather=gather)
        for w in range(args.warmup):
            pic.pic_step(ctx, st, box, -1.0, -1e-4, dt, **kw)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            if resort and (i + args.warmup) % args.resort == 0:
                pic.pic_sort(ctx, st, tiled=tiled, sync=False)
            pic.pic_step(ctx, st, box, -1.0, -1e-4, dt, sync=False, **kw)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        msp = e0.elapsed_time(e1) / args.steps
        nb2 = (n_before + pic.pic_sync(ctx, st)) / 2
        out[mode]["ms_pipelined"] = msp
        out[mode]["frac_of_hbm_peak_pipelined"] = BYTES_PER_PARTICLE * nb2 / (msp / 1e3) / 1e9 / peak
        del st
    for a, b in (("push_deposit", "push_deposit_noclock"),
                 ("push_deposit_resort", "push_deposit_resort_noclock"),
                 ("push_deposit_fast_resort", "push_deposit_fast_resort_noclock"),
                 ("push_deposit_esk3_resort", "push_deposit_esk3_resort_noclock")):
        if a in out and b in out:   # GpuClock tally in that kernel vs the same kernel without it
            out[f"gpuclock_overhead_{a}"] = out[a]["ms_pipelined"] / out[b]["ms_pipelined"] - 1.0
    out["peak_gbs"] = peak
    out["peak_source"] = peak_src
    print(json.dumps(out))


if __name__ == "__main__":
    main()
