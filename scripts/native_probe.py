"""Native-size step time (C2 at 801 k particles, C1 at 131 k) across rank
counts / cost kinds, with the device span of each step's kernels, to see
whether the native loop is host- or GPU-bound."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2104_11385_b200.workload import Simulation  # noqa: E402

dev = torch.device("cuda:0")
out = {}
for ranks in (1, 8, 24):
    for cost in ("heuristic", "gpuclock"):
        spec, sc = bench.c2_spec(ranks, 420, cost)
        pos0, kick0 = bench.base_particles(spec)
        for timed in (False, True):
            sim = Simulation(sc, spec.policy, spec.build_provider(), device=dev,
                             positions=torch.from_numpy(pos0).to(dev),
                             kick=torch.from_numpy(kick0).to(dev), time_kernels=timed)
            sim.run(0, 20)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            sim.run(20, 420)
            e1.record()
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            r = sim.result() if timed else None
            out[f"r{ranks}_{cost}_{'timed' if timed else 'plain'}"] = {
                "us_per_step": 1e3 * e0.elapsed_time(e1) / 400, "wall_us_per_step": 1e6 * wall / 400,
                "kernel_us_mean": None if r is None else float(1e3 * np.mean(r.kernel_ms[20:420]))}
            sim.close()
c1 = bench.c1_uniform(dev)
out["c1"] = {k: c1[k] for k in ("gpu_us_per_step",)}
print(json.dumps(out, indent=1))
