"""CPU tests of the reference-API mirror: host-side pieces (scenario
sampling, kick, mappings, config parsing, perfmodel) against the oracle."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import lbsim_oracle as O

G = Path(__file__).resolve().parent / "golden"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def P():
    import paper_2104_11385_b200 as P
    return P


@pytest.mark.parametrize("name", ["mini", "tight-memory", "default"])
def test_presets_sample_reference_positions(P, name):
    runs = json.loads((G / "runs.json").read_text())
    key = {"mini": "mini", "tight-memory": "tight", "default": "default_short"}[name]
    from paper_2104_11385_b200.workload import kick_velocities, sample_blob
    cfg = P.load_spec(name).scenario
    pos = sample_blob(cfg)
    assert sha(pos) == runs[key]["init_pos_sha"]
    assert pos.shape[0] == runs[key]["n_init"]
    kv = kick_velocities(pos, cfg)
    want = O.kick_velocities(pos, cfg.blob.center, cfg.kick.speed, cfg.kick.drift, cfg.seed)
    assert np.array_equal(kv, want)


def test_frozen_monte_carlo_count(P):
    from paper_2104_11385_b200.workload import sample_blob
    cfg = P.ScenarioConfig(scenario_id="mc", domain_extent=(240, 240), box_size=16,
                           n_ranks=4, blob=P.BlobSpec((120.0, 120.0), 40.0, 0.0, 4.0),
                           kick=P.KickSpec(5, 0.1), total_steps=10, seed=4242)
    assert sample_blob(cfg).shape[0] == 20104


def test_balancer_api_known_answers(P):
    cv = lambda v: P.CostVector(values=np.asarray(v, float))  # noqa: E731
    dm = lambda o, r: P.DistributionMapping(owner=np.asarray(o), n_ranks=r)  # noqa: E731
    assert P.efficiency(cv([18, 0, 0, 12]), dm([0, 1, 1, 0], 2)) == 0.5
    assert P.efficiency_flagged(cv([0, 0]), dm([0, 1], 2)) == (1.0, True)
    m = P.knapsack_assign(cv([3, 3, 2, 2, 2]), 2)
    from paper_2104_11385_b200.balancer import rank_loads
    assert rank_loads(cv([3, 3, 2, 2, 2]), m).max() == 6.0
    with pytest.raises(ValueError, match="cap"):
        P.knapsack_assign(cv([1, 2, 3]), 2, cap_factor=0.0)
    with pytest.raises(ValueError, match="length"):
        P.efficiency(cv([1, 2, 3]), dm([0, 1], 2))
    with pytest.raises(ValueError, match="curve"):
        from paper_2104_11385_b200.balancer import BalancePolicy, Strategy
        P.attempt_rebalance(cv([1, 2]), dm([0, 1], 2),
                            BalancePolicy(strategy=Strategy.SFC), 0)
    ba = P.build_box_array((64, 64), 16)
    assert P.morton_order(ba).tolist() == O.morton_order(4, 4).tolist()
    assert P.morton_index((3, 5)) == 39
    own = P.sfc_assign(cv(np.arange(16.0)), P.morton_order(ba), 3).owner
    assert own.tolist() == O.sfc_assign(np.arange(16.0), O.morton_order(4, 4), 3).tolist()
    opt = P.sfc_assign_optimal(cv(np.arange(16.0)), P.morton_order(ba), 3).owner
    assert opt.tolist() == O.sfc_assign_optimal(np.arange(16.0), O.morton_order(4, 4), 3).tolist()


def test_measured_cost_api(P):
    f = np.load(G / "measured.npz")
    work = np.linspace(1.0, 1000.0, 900)
    got = P.measured_cost(work, P.MeasurementConfig(noise_amplitude=0.05, seed=7), step=0)
    assert np.array_equal(got.values, f["7_0_900"])


def test_config_errors_name_the_field(P):
    from paper_2104_11385_b200.scenarios import spec_from_dict
    with pytest.raises(P.ConfigError, match="domain"):
        spec_from_dict({"scenario_id": "x"})
    with pytest.raises(P.ConfigError, match="box_size 7 does not divide the z-extent"):
        P.build_box_array((64, 64), 7)
    with pytest.raises(P.ConfigError):
        P.make_provider("nvtx")
    assert P.make_provider("GpuClock").kind == "gpuclock"
    assert P.make_provider("Timers").kind == "timers"
    assert P.make_provider("CUPTI").kind == "cupti" and P.make_provider("cupti").device_kind == 5
    s = P.apply_overrides(P.load_spec("mini"), policy="none")
    assert s.policy.interval == s.scenario.total_steps + 1
    s = P.apply_overrides(P.load_spec("mini"), policy="static", ranks=4)
    assert s.policy.static_step == 0 and s.scenario.n_ranks == 4


def test_gpuclock_provider_forms(P):
    """GpuClock cost forms: raw = the tally; calibrated = the tallies summed
    over the LB window, scaled to the heuristic's particle units, + the
    per-box cell work (the same operations as lbx_runtime.cpp's lb_step)."""
    clk = np.array([0, 1000, 3000, 0, 6000], dtype=np.uint64)
    counts = np.array([0, 10, 30, 0, 60], dtype=np.int64)
    cells = np.full(5, 1024.0)
    raw = P.make_provider("gpuclock-raw")
    assert raw.kind == "gpuclock-raw" and raw.clock_mode == 0
    assert raw.assess(counts, cells, None, 0, clock=clk).values.tolist() == clk.tolist()
    cal = P.make_provider("gpuclock")
    assert cal.clock_mode == 1
    v = cal.assess(counts, cells, None, 0, clock=clk).values
    scale = 0.75 * 100.0 / 10000.0
    assert v.tolist() == [c * scale + 0.25 * 1024.0 for c in clk.astype(float)]
    assert abs(v.sum() - (0.75 * counts.sum() + 0.25 * cells.sum())) < 1e-9
    # second step of the window: tallies and particles accumulate
    clk2 = np.array([0, 3000, 1000, 0, 6000], dtype=np.uint64)
    v2 = cal.assess(counts, cells, None, 1, clock=clk2).values
    acc = (clk + clk2).astype(float)
    scale2 = 0.75 * (200.0 / 2.0) / acc.sum()
    assert v2.tolist() == [c * scale2 + 0.25 * 1024.0 for c in acc]
    cal.reset_window()
    assert cal.assess(counts, cells, None, 2, clock=clk).values.tolist() == v.tolist()
    with pytest.raises(ValueError, match="clock"):
        cal.assess(counts, cells, None, 0)
    with pytest.raises(P.ConfigError):
        P.GpuClockProvider("fast")


def test_perfmodel(P):
    assert abs(P.max_speedup(1 / 6.2, 0.91) - 5.261) < 1e-3
    m = P.fit_scaling([(n, 3.0 * n ** -0.9) for n in (1, 2, 4, 8)])
    assert abs(m.exponent - 0.9) < 1e-12


def test_resolve_costs_matches_oracle(P):
    from paper_2104_11385_b200.workload import resolve_costs
    from tests.scenario_util import preset_doc
    for name in ("mini", "tight-memory", "default"):
        cm = resolve_costs(P.load_spec(name).scenario)
        want = O.resolve_costs(O.config_from_doc(preset_doc(name)))
        assert (cm.comm_per_face, cm.gather, cm.redistribute_per_particle,
                cm.redistribute_latency) == want
