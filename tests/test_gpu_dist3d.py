"""Multi-GPU 3D (three_d.Distributed3D) with its real kernels
(lbx_push_step_3d_exchange, lbx_partition_3d, group / unpack / hole fill):
`world` ranks as threads sharing cuda:0 through parallel.ThreadComm must
reproduce the single-GPU Simulation3D run -- per-box counts, cost trace,
mappings -- and its particle multiset."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CFG = dict(scenario_id="c4-threads", domain_extent=(64, 64, 32), box_size=16, n_ranks=2,
           center=(20.0, 32.0, 16.0), core_radius=10.0, edge_scale=2.0,
           particles_per_cell=3.0, kick_step=2, kick_speed=0.9, kick_drift=0.3,
           total_steps=30, seed=3)


def rows(a):
    a = np.asarray(a)
    return a[np.lexsort(a.T[::-1])]


def run_threads(cfg, pol, cost, world, replicas=1):
    from paper_2104_11385_b200.cost import make_provider
    from paper_2104_11385_b200.parallel import ThreadComm
    from paper_2104_11385_b200.three_d import Distributed3D
    shared = ThreadComm.shared(world)
    outs, errs = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            sim = Distributed3D(cfg, pol, make_provider(cost), comm=ThreadComm(shared, r),
                                device="cuda:0", record_counts=True, replicas=replicas)
            sim.run()
            outs[r] = (dict(sim.out), sim.local_state(), sim.moved.copy(),
                       int(sim.souts.n_adoptions), sim.engine.launches)
            sim.close()
        except Exception as e:
            errs.append(e)
            shared["bar"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return outs


@pytest.mark.parametrize("world,strategy,interval,replicas",
                         [(2, "knapsack", 4, 1), (3, "sfc", 5, 2), (4, "knapsack", 3, 1)])
def test_distributed3d_threads_match_simulation3d(world, strategy, interval, replicas):
    from paper_2104_11385_b200.balancer import BalancePolicy, Strategy
    from paper_2104_11385_b200.cost import make_provider
    from paper_2104_11385_b200.three_d import (Scenario3D, Simulation3D, kick_velocities_3d,
                                               sample_blob_3d)
    cfg = Scenario3D(**dict(CFG, n_ranks=world))
    pol = BalancePolicy(strategy=Strategy(strategy), interval=interval)
    outs = run_threads(cfg, pol, "heuristic", world, replicas)
    pos0 = sample_blob_3d(cfg)
    kick = kick_velocities_3d(pos0, cfg)
    ref = Simulation3D(cfg, pol, make_provider("heuristic"), record_counts=True,
                       positions=torch.from_numpy(np.tile(pos0, (replicas, 1))).cuda(),
                       kick=np.tile(kick, (replicas, 1)))
    ref.run()
    nad = int(ref.souts.n_adoptions)
    assert nad >= 1
    for o, _, _, n_ad, launches in outs:
        assert n_ad == nad and launches > 0
        for k in ("count_trace", "cost_trace", "eff_before", "eff_after", "adopted", "walltime"):
            assert np.array_equal(o[k], ref.out[k]), k
        assert np.array_equal(o["adopt_owners"][:nad], ref.out["adopt_owners"][:nad])
    assert sum(m.sum() for _, _, m, _, _ in outs) > 0
    gp = np.concatenate([s[0] for _, s, _, _, _ in outs])
    gv = np.concatenate([s[1] for _, s, _, _, _ in outs])
    rp, rv = ref.state()
    assert np.array_equal(rows(np.column_stack([gp, gv])), rows(np.column_stack([rp, rv])))
    ref.close()


def test_distributed3d_gpuclock_counts_match():
    """GpuClock costs are measured per rank and all-reduced; the per-box
    counts stay exact (every rank runs the same mapping decisions)."""
    from paper_2104_11385_b200.balancer import BalancePolicy, Strategy
    from paper_2104_11385_b200.three_d import Scenario3D
    cfg = Scenario3D(**dict(CFG, n_ranks=2))
    outs = run_threads(cfg, BalancePolicy(strategy=Strategy.KNAPSACK, interval=5), "gpuclock", 2)
    a, b = outs[0][0], outs[1][0]
    assert np.array_equal(a["count_trace"], b["count_trace"])
    assert np.array_equal(a["cost_trace"], b["cost_trace"])
    assert outs[0][3] == outs[1][3]
