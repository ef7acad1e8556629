"""The benchmark's replica-tiled C2 workload is checkable at full size:
every replica evolves identically, so per-box counts must be exactly R times
the oracle's counts on the base set, every step."""
import numpy as np
import pytest

from oracle import lbsim_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("R,steps,cost", [(3, 12, "heuristic"), (128, 4, "gpuclock")])
def test_replica_counts_are_R_times_oracle(R, steps, cost):
    import bench
    from paper_2104_11385_b200.workload import Simulation
    spec, sc = bench.c2_spec(1, steps, cost)
    pos0, kick0 = bench.base_particles(spec)
    dev = torch.device("cuda:0")
    pos = torch.from_numpy(pos0).to(dev).repeat(R, 1)
    kick = torch.from_numpy(kick0).to(dev).repeat(R, 1)
    sim = Simulation(sc, spec.policy, spec.build_provider(), device=dev, positions=pos,
                     kick=kick, record_counts=True)
    sim.run()
    res = sim.result()
    p, v = pos0, kick0
    nb = 30
    for s in range(steps):
        p, v = O.advance_particles(p, v, 960.0, 960.0)
        c = O.bin_particles(p, 32.0, nb, nb)
        assert np.array_equal(res.count_trace[s], R * c), s
        assert res.n_alive[s] == R * p.shape[0]
    if cost == "heuristic":
        assert np.array_equal(res.cost_trace[-1],
                              O.heuristic_cost(R * c, np.full(nb * nb, 1024), 0.75, 0.25))
    sim.close()
