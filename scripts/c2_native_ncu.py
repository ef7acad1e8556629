"""A few native-loop steps of C2 at native size (for an ncu launch list)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2104_11385_b200.workload import Simulation  # noqa: E402

dev = torch.device("cuda:0")
spec, sc = bench.c2_spec(1, 40, sys.argv[1] if len(sys.argv) > 1 else "gpuclock")
pos0, kick0 = bench.base_particles(spec)
sim = Simulation(sc, spec.policy, spec.build_provider(), device=dev,
                 positions=torch.from_numpy(pos0).to(dev), kick=torch.from_numpy(kick0).to(dev))
sim.run(0, 40)
torch.cuda.synchronize()
sim.close()
