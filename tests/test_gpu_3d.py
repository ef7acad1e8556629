"""3D extension (config C4; parity unpinned -- the reference is 2D): the 3D
fused kernel + 3D LB host step against the oracle's 3D restatement."""
import numpy as np
import pytest

from oracle import lbsim_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_3d_run_counts_and_state_exact():
    from paper_2104_11385_b200.balancer import BalancePolicy, Strategy
    from paper_2104_11385_b200.cost import make_provider
    from paper_2104_11385_b200.three_d import (Scenario3D, Simulation3D, kick_velocities_3d,
                                               sample_blob_3d)
    cfg = Scenario3D("c4-small", (64, 64, 32), 16, 4, (20.0, 32.0, 16.0), 10.0, 2.0, 3.0,
                     kick_step=2, kick_speed=0.9, kick_drift=0.3, total_steps=20, seed=3)
    pol = BalancePolicy(strategy=Strategy.SFC, interval=5)
    sim = Simulation3D(cfg, pol, make_provider("heuristic"), record_counts=True)
    sim.run()
    pos = sample_blob_3d(cfg)
    vel = np.zeros_like(pos)
    kick = kick_velocities_3d(pos, cfg)
    for s in range(cfg.total_steps):
        if s == cfg.kick_step:
            vel = kick
        pos, vel = O.advance_particles_3d(pos, vel, cfg.domain_extent)
        c = O.bin_particles_3d(pos, 16.0, cfg.grid)
        assert np.array_equal(sim.out["count_trace"][s], c), s
    gp, gv = sim.state()
    assert np.array_equal(gp, pos) and np.array_equal(gv, vel)
    assert sim.out["attempted"].sum() == 4
    sim.close()
