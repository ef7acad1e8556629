"""Native-size (801k) and C2x128 step times of the current libLBX build
(LBX_VARIANT selects a tuning build): us/step of the native loop and the
fused kernel's mean ms at x128."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2104_11385_b200.workload import Simulation  # noqa: E402

dev = torch.device("cuda:0")
out = {"variant": os.environ.get("LBX_VARIANT", "")}
for cost in ("heuristic", "gpuclock"):
    spec, sc = bench.c2_spec(1, 420, cost)
    pos0, kick0 = bench.base_particles(spec)
    sim = Simulation(sc, spec.policy, spec.build_provider(), device=dev,
                     positions=torch.from_numpy(pos0).to(dev),
                     kick=torch.from_numpy(kick0).to(dev), time_kernels=True)
    sim.run(0, 20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.run(20, 420)
    e1.record()
    torch.cuda.synchronize()
    r = sim.result()
    out[f"native_{cost}_us_per_step"] = 1e3 * e0.elapsed_time(e1) / 400
    out[f"native_{cost}_kernel_us"] = float(1e3 * np.mean(r.kernel_ms[20:420]))
    sim.close()
spec, sc = bench.c2_spec(1, 25, "gpuclock")
pos0, kick0 = bench.base_particles(spec)
R = 128
sim = Simulation(sc, spec.policy, spec.build_provider(), device=dev,
                 positions=torch.from_numpy(pos0).to(dev).repeat(R, 1),
                 kick=torch.from_numpy(kick0).to(dev).repeat(R, 1), time_kernels=True)
sim.run(0, 25)
torch.cuda.synchronize()
out["x128_kernel_ms"] = float(np.mean(sim.result().kernel_ms[5:25]))
sim.close()
print(json.dumps(out))
