"""Native-size loop time of the resident kernel (C2 801 k at 1/8/24 ranks,
C1), for A/B of libLBX build variants (LBX_VARIANT)."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2104_11385_b200.workload import Simulation  # noqa: E402

dev = torch.device("cuda:0")
out = {"variant": os.environ.get("LBX_VARIANT", "")}
for ranks, cost in ((1, "heuristic"), (8, "gpuclock"), (24, "heuristic")):
    spec, sc = bench.c2_spec(ranks, 420, cost)
    pos0, kick0 = bench.base_particles(spec)
    sim = Simulation(sc, spec.policy, spec.build_provider(), device=dev,
                     positions=torch.from_numpy(pos0).to(dev), kick=torch.from_numpy(kick0).to(dev))
    sim.run(0, 20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.run(20, 420)
    e1.record()
    torch.cuda.synchronize()
    out[f"c2_r{ranks}_{cost}"] = round(1e3 * e0.elapsed_time(e1) / 400, 2)
    sim.close()
out["c1"] = round(bench.c1_uniform(torch.device("cuda:0"))["gpu_us_per_step"], 2)
print(json.dumps(out), flush=True)
