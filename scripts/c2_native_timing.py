"""C2 at native size: native-loop step time vs the device span of each step's
kernels (time_kernels=True), to see whether the loop is host- or GPU-bound."""
import json
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2104_11385_b200.workload import Simulation  # noqa: E402

dev = torch.device("cuda:0")
out = {}
for cost in sys.argv[2].split(",") if len(sys.argv) > 2 else ("gpuclock", "heuristic"):
    spec, sc = bench.c2_spec(int(sys.argv[1]) if len(sys.argv) > 1 else 1, 420, cost)
    pos0, kick0 = bench.base_particles(spec)
    for timed in (False, True):
        sim = Simulation(sc, spec.policy, spec.build_provider(), device=dev,
                         positions=torch.from_numpy(pos0).to(dev),
                         kick=torch.from_numpy(kick0).to(dev), time_kernels=timed)
        sim.run(0, 20)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sim.run(20, 420)
        e1.record()
        torch.cuda.synchronize()
        r = sim.result() if timed else None
        out[f"{cost}_{'timed' if timed else 'plain'}"] = {
            "us_per_step": 1e3 * e0.elapsed_time(e1) / 400,
            "kernel_us_mean": None if r is None else float(1e3 * np.mean(r.kernel_ms[20:420]))}
        sim.close()
print(json.dumps(out))
