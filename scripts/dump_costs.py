"""Cost vectors of a native-size C2 run at its LB attempt steps (for host
knapsack timing off the GPU box): gpurun_out/c2_costs_<ranks>_<cost>.npz."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2104_11385_b200.workload import Simulation  # noqa: E402

for ranks, cost in ((8, "gpuclock"), (24, "gpuclock"), (8, "heuristic")):
    spec, sc = bench.c2_spec(ranks, 420, cost)
    pos0, kick0 = bench.base_particles(spec)
    sim = Simulation(sc, spec.policy, spec.build_provider(), device="cuda:0",
                     positions=torch.from_numpy(pos0).cuda(), kick=torch.from_numpy(kick0).cuda())
    sim.run(0, 420)
    r = sim.result()
    sim.close()
    att = np.arange(0, len(r.metrics), spec.policy.interval)
    np.savez(f"gpurun_out/c2_costs_{ranks}_{cost}.npz", steps=att, cost=r.cost_trace[att],
             owner0=r.initial_owner)
    print(ranks, cost, len(att), r.summary["adoption_count"])
