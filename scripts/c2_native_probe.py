import sys, torch
sys.path.insert(0, "/root/repo")
import bench
from dataclasses import replace
from paper_2104_11385_b200.workload import Simulation
dev = torch.device("cuda:0")
spec, sc = bench.c2_spec(1, 10, "gpuclock")
pos0, kick0 = bench.base_particles(spec)
sc1 = replace(sc, total_steps=60)
sim = Simulation(sc1, spec.policy, spec.build_provider(), device=dev, positions=torch.from_numpy(pos0).to(dev), kick=torch.from_numpy(kick0).to(dev))
sim.run(0, 60)
torch.cuda.synchronize()
print("ok")
