"""Run-level properties of `run_simulation` on the GPU native loop -- the
reference's `TestRunSimulation` checks (`test_workload.py:206-287`) restated
for this package: determinism, the none / static / dynamic policies, exact
walltime decomposition, efficiency recomputable from the emitted trace,
zero-overhead walltime == sum of max rank compute, OOM halting."""
from dataclasses import replace

import numpy as np
import pytest

import paper_2104_11385_b200 as P

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def small(**overrides):
    base = dict(scenario_id="small", domain_extent=(96, 96), box_size=16, n_ranks=4,
                blob=P.BlobSpec(center=(48.0, 48.0), core_radius=16.0, edge_scale=2.0,
                                particles_per_cell=6.0),
                kick=P.KickSpec(step=3, speed=0.4, drift=0.1), total_steps=40, seed=21)
    base.update(overrides)
    return P.ScenarioConfig(**base)


def run(cfg, provider=None, **policy):
    return P.run_simulation(cfg, P.BalancePolicy(**policy),
                            provider or P.make_provider("heuristic"))


def test_runs_are_deterministic():
    a, b = run(small(), interval=5), run(small(), interval=5)
    assert a.metrics == b.metrics and a.summary == b.summary
    assert np.array_equal(a.cost_trace, b.cost_trace)


def test_no_balancing_keeps_the_initial_mapping():
    cfg = small()
    res = run(cfg, interval=cfg.total_steps + 1)
    assert res.summary["adoption_count"] == 0 and res.summary["attempt_count"] == 0
    assert not res.adoption_snapshots
    assert all(m.efficiency_before == m.efficiency_after for m in res.metrics)


def test_dynamic_balancing_beats_none():
    cfg = small(total_steps=60)
    dyn, none = run(cfg, interval=5), run(cfg, interval=cfg.total_steps + 1)
    assert dyn.summary["mean_efficiency"] > none.summary["mean_efficiency"]
    assert dyn.summary["adoption_count"] > 0


def test_static_policy_attempts_once():
    res = run(small(total_steps=30), interval=31, static_step=0)
    assert res.summary["attempt_count"] == 1 and res.summary["policy"] == "static"


def test_walltime_is_the_sum_of_its_columns():
    res = run(small(), interval=5)
    assert 0.0 < res.summary["mean_efficiency"] <= 1.0
    for m in res.metrics:
        assert m.walltime == m.compute_max + m.comm_max + m.gather + m.redistribute


def test_efficiency_series_recomputes_from_the_trace():
    cfg = small(total_steps=25)
    res = run(cfg, interval=99)
    mapping = P.DistributionMapping(owner=res.initial_owner, n_ranks=cfg.n_ranks)
    for m, row in zip(res.metrics, res.cost_trace):
        value, _ = P.efficiency_flagged(P.CostVector(values=row), mapping)
        assert m.efficiency_before == value


def test_zero_overheads_make_walltime_the_max_rank_compute():
    free = P.CostModel(comm_per_face=0.0, gather=0.0, redistribute_per_particle=0.0,
                       redistribute_latency=0.0)
    cfg = small(costs=free, total_steps=30)
    res = run(cfg, interval=99)
    owner = res.initial_owner
    c_max = sum(np.bincount(owner, weights=row, minlength=cfg.n_ranks).max()
                for row in res.cost_trace)
    assert res.summary["total_walltime"] == pytest.approx(c_max, rel=1e-12)


def test_capacity_overflow_halts_with_a_completion_fraction():
    n0 = P.init_scenario(small()).n_particles
    cfg = small(capacity_particles=max(1, n0 // 8))
    res = run(cfg, interval=cfg.total_steps + 1)
    assert res.summary["oom"] and res.metrics[-1].oom
    assert res.summary["completed_steps"] < cfg.total_steps
    assert 0.0 < res.summary["completion_fraction"] < 1.0


@pytest.mark.parametrize("kind", ["measured", "gpuclock"])
def test_device_and_modelled_timers_keep_the_particles(kind):
    """The cost strategy only changes costs and mappings, never the particle
    state: final particles equal the heuristic run's."""
    cfg = replace(small(), total_steps=30)
    ref = run(cfg, interval=5)
    res = run(cfg, P.make_provider(kind, seed=cfg.seed), interval=5)
    assert res.summary["final_particles"] == ref.summary["final_particles"]
    a, b = ref.final_state.to_numpy(), res.final_state.to_numpy()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
