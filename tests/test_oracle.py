"""Pin the CPU oracle against fixtures produced by the real reference.

These run on CPU (no GPU): they are what makes the oracle trustworthy as the
checker for the CUDA path.
"""
import hashlib
import importlib.util
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import lbsim_oracle as O

G = Path(__file__).resolve().parent / "golden"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def runs():
    return json.loads((G / "runs.json").read_text())


def test_kernels_match_reference_fixture():
    f = np.load(G / "kernels.npz")
    for tag in "abcd":
        e = float(f[f"{tag}_extent"])
        p, v = O.advance_particles(f[f"{tag}_pos"], f[f"{tag}_vel"], e, e)
        assert np.array_equal(p, f[f"{tag}_out_pos"])
        assert np.array_equal(v, f[f"{tag}_out_vel"])
        assert np.array_equal(O.bin_particles(p, e / 8, 8, 8), f[f"{tag}_bins"])
    p, v = f["chain_pos"], f["chain_vel"]
    for _ in range(25):
        p, v = O.advance_particles(p, v, 64.0, 64.0)
    assert np.array_equal(p, f["chain_out_pos"]) and np.array_equal(v, f["chain_out_vel"])


def test_known_answers_from_reference_tests():
    # test_kernels.py:36-41
    pos = np.array([[1.0, 1.0], [2.0, 2.0], [63.5, 63.5], [3.0, 3.0]])
    vel = np.array([[0.1, 0.0], [0.0, 0.0], [1.0, 1.0], [0.0, -0.5]])
    p, _ = O.advance_particles(pos, vel, 64.0, 64.0)
    assert np.array_equal(p, [[1.1, 1.0], [2.0, 2.0], [3.0, 2.5]])
    # test_cost.py:24-36
    assert O.heuristic_cost([18, 0, 0, 12], [0, 0, 0, 0], 1.0, 0.0).tolist() == [18, 0, 0, 12]
    assert O.heuristic_cost([1000, 1024], [4, 0], 1.0, 24.75).tolist()[0] == 1099.0
    # test_balancer.py:37-50
    assert O.efficiency_flagged([18, 0, 0, 12], [0, 1, 1, 0], 2)[0] == 0.5
    assert O.efficiency_flagged([5, 3, 3, 1], [0, 0, 1, 1], 2)[0] == 0.75
    assert O.efficiency_flagged([0, 0], [0, 1], 2) == (1.0, True)
    # test_balancer.py:92-97: swap refinement beats plain LPT
    own = O.knapsack_assign([3, 3, 2, 2, 2], 2)
    assert O.rank_loads([3, 3, 2, 2, 2], own, 2).max() == 6.0
    # test_decomposition.py:77-79
    assert O.morton_code(3, 5) == 39


def test_balancer_matches_reference_fixture():
    f = np.load(G / "balancer.npz")
    meta = f["meta"]
    for i, (nbz, nbx, R, cap, e_ks, e_sf) in enumerate(meta):
        R = int(R)
        c = f[f"c{i}"]
        curve = O.morton_order(int(nbz), int(nbx))
        assert np.array_equal(curve, f[f"m{i}"])
        if f[f"k{i}"][0] >= 0:
            ks = O.knapsack_assign(c, R, cap)
            assert np.array_equal(ks, f[f"k{i}"]), i
            assert O.efficiency_flagged(c, ks, R)[0] == e_ks
        else:
            with pytest.raises(ValueError):
                O.knapsack_assign(c, R, cap)
        sf = O.sfc_assign(c, curve, R)
        assert np.array_equal(sf, f[f"s{i}"]), i
        assert O.efficiency_flagged(c, sf, R)[0] == e_sf
    for R in (8, 24):
        assert np.array_equal(O.knapsack_assign(f["big_c"], R), f[f"big_k{R}"])
        assert np.array_equal(O.sfc_assign(f["big_c"], f["big_curve"], R), f[f"big_s{R}"])


def test_measured_matches_reference_fixture():
    f = np.load(G / "measured.npz")
    amps = {"7_0_900": 0.05, "11_123_225": 0.05, "13_599_900": 0.2, "0_5_17": 0.5,
            f"{2**40+3}_{2**33}_64": 0.05}
    for key, amp in amps.items():
        seed, step, n = (int(x) for x in key.split("_"))
        got = O.measured_cost(np.linspace(1.0, 1000.0, n), amp, seed, step)
        assert np.array_equal(got, f[key]), key


RUN_CASES = ["mini", "mini_none", "mini_static", "mini_sfc", "mini_measured",
             "mini_instrumented", "tight", "tight_none", "c1", "small", "leaky"]


def load_case(runs, name):
    from tests.scenario_util import case_config
    return case_config(runs, name)


@pytest.mark.parametrize("name", RUN_CASES)
def test_whole_run_matches_reference(runs, name):
    cfg = load_case(runs, name)
    res = O.run_simulation(cfg, record_counts=True)
    ref = runs[name]
    for k, v in ref["metrics"].items():
        assert res["metrics"][k].tolist() == v, (name, k)
    assert sha(res["cost_trace"]) == ref["cost_trace_sha"]
    assert sha(res["count_trace"].astype(np.int64)) == ref["count_trace_sha"]
    assert res["initial_owner"].tolist() == ref["initial_owner"]
    assert [[s, o.tolist()] for s, o in res["snapshots"]] == ref["snapshots"]
    for k in ("completed_steps", "total_walltime", "mean_efficiency", "adoption_count",
              "attempt_count", "oom", "final_particles", "completion_fraction"):
        assert res["summary"][k] == ref["summary"][k], (name, k)
    assert sha(res["final_pos"]) == ref["final_pos_sha"]
    assert sha(res["final_vel"]) == ref["final_vel_sha"]


def test_frozen_monte_carlo_count():
    # test_workload.py:52-67: frozen sampled count 20104
    pos, _ = O.init_scenario((240, 240), 16, (120.0, 120.0), 40.0, 0.0, 4.0, 4242)
    assert pos.shape[0] == 20104


def test_compiled_reference_kernels_agree_with_oracle():
    """oracle/_ref holds the reference's own Cython kernels (compiled by
    oracle/Makefile); they must agree bit-for-bit with the restatement."""
    ref_dir = Path(__file__).resolve().parent.parent / "oracle" / "_ref"
    cands = list(ref_dir.glob("_kernels*.so")) if ref_dir.exists() else []
    if not cands:
        pytest.skip("oracle/_ref not built (run `make -C oracle`)")
    spec = importlib.util.spec_from_file_location("_kernels", cands[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    f = np.load(G / "kernels.npz")
    for tag in "abcd":
        e = float(f[f"{tag}_extent"])
        p, v = mod.advance_particles(f[f"{tag}_pos"], f[f"{tag}_vel"], e, e)
        assert np.array_equal(p, f[f"{tag}_out_pos"])
        assert np.array_equal(v, f[f"{tag}_out_vel"])
        assert np.array_equal(mod.bin_particles(p, e / 8, 8, 8), f[f"{tag}_bins"])
