"""Multi-rank 3D protocol (three_d.Distributed3D) on CPU with gloo, world
size 2 and 3: global per-box counts, replicated 3D LB decisions and
adoption-time migration must reproduce a single-process run of the oracle's
3D step with the same host LB object exactly, and the particle multiset."""
import ctypes as C

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import lbsim_oracle as O
from tests.dist_util import free_port
from tests.dist3d_util import run_rank3d

CFG = dict(scenario_id="c4-gloo", domain_extent=(64, 64, 32), box_size=16, n_ranks=2,
           center=(20.0, 32.0, 16.0), core_radius=10.0, edge_scale=2.0,
           particles_per_cell=1.0, kick_step=2, kick_speed=0.9, kick_drift=0.3,
           total_steps=24, seed=3)


def single_process(cfg_kw, pol_kw):
    from paper_2104_11385_b200 import _lib
    from paper_2104_11385_b200.balancer import BalancePolicy, Strategy
    from paper_2104_11385_b200.cost import make_provider
    from paper_2104_11385_b200.three_d import (Scenario3D, initial_owner_3d, kick_velocities_3d,
                                               lb_config_3d, sample_blob_3d)
    cfg = Scenario3D(**cfg_kw)
    pol = BalancePolicy(strategy=Strategy(pol_kw["strategy"]), interval=pol_kw["interval"])
    conf, _, _ = lb_config_3d(cfg, pol, make_provider("heuristic"))
    pos = sample_blob_3d(cfg)
    own = np.ascontiguousarray(initial_owner_3d(cfg, pos), dtype=np.int64)
    h = C.c_void_p()
    _lib.check(_lib.lib.lbx_lb_create(C.byref(h), C.byref(conf), _lib.ptr(own)))
    T, nb = cfg.total_steps, cfg.n_boxes
    o = {k: np.zeros(T) for k in ("eff_before", "eff_after", "compute_max", "comm_max",
                                  "gather", "redistribute", "walltime")}
    for k in ("adopted", "attempted", "oom"):
        o[k] = np.zeros(T, dtype=np.uint8)
    o["max_rank_particles"] = np.zeros(T, dtype=np.int64)
    o["n_alive"] = np.zeros(T, dtype=np.int64)
    o["cost_trace"] = np.zeros((T, nb))
    o["count_trace"] = np.zeros((T, nb), dtype=np.int64)
    o["adopt_steps"] = np.zeros(T, dtype=np.int64)
    o["adopt_owners"] = np.zeros((T, nb), dtype=np.int64)
    so = _lib.SimOutputs(*(_lib.ptr(o.get(k)) for k in (
        "eff_before", "eff_after", "adopted", "attempted", "compute_max", "comm_max", "gather",
        "redistribute", "walltime", "max_rank_particles", "oom", "n_alive", "cost_trace",
        "count_trace", "clock_trace", "owner", "adopt_steps", "adopt_owners")), None, 0, 0, 0)
    vel = np.zeros_like(pos)
    kick = kick_velocities_3d(pos, cfg)
    a, hl = C.c_int32(), C.c_int32()
    for s in range(T):
        if s == cfg.kick_step:
            vel = kick
        pos, vel = O.advance_particles_3d(pos, vel, cfg.domain_extent)
        counts = O.bin_particles_3d(pos, float(cfg.box_size), cfg.grid)
        _lib.check(_lib.lib.lbx_lb_step(h, s, _lib.ptr(counts), None, int(counts.sum()),
                                        C.byref(so), C.byref(a), C.byref(hl)))
    _lib.lib.lbx_lb_destroy(h)
    o["adopt_owners"] = o["adopt_owners"][:int(so.n_adoptions)]
    return o, pos, vel


def rows(a):
    a = np.asarray(a)
    return a[np.lexsort(a.T[::-1])]


@pytest.mark.parametrize("world,strategy,interval", [(2, "knapsack", 4), (3, "sfc", 5)])
def test_distributed3d_matches_single_process(tmp_path, world, strategy, interval):
    cfg_kw = dict(CFG, n_ranks=world)
    pol_kw = {"strategy": strategy, "interval": interval}
    mp.spawn(run_rank3d, args=(world, free_port(), cfg_kw, pol_kw, str(tmp_path)), nprocs=world)
    ref, pos, vel = single_process(cfg_kw, pol_kw)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    assert len(ref["adopt_owners"]) >= 1   # the run migrates at least once
    for o in outs:
        for k in ("count_trace", "cost_trace", "eff_before", "eff_after", "adopted", "walltime",
                  "adopt_owners"):
            assert np.array_equal(o[k], ref[k]), k
    assert sum(o["moved"].sum() for o in outs) > 0
    gp = np.concatenate([o["pos"] for o in outs])
    gv = np.concatenate([o["vel"] for o in outs])
    assert np.array_equal(rows(np.column_stack([gp, gv])), rows(np.column_stack([pos, vel])))
