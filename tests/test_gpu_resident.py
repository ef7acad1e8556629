"""The resident multi-step kernel (lbx_resident.cu) against the per-step
kernels: every output of the native loop and the final particle state are
identical, over split runs whose boundaries fall before, at and after the
kick, for each cost form the resident path serves."""
import hashlib

import numpy as np
import pytest

from tests.test_gpu_runs import runs, spec_for  # noqa: F401  (fixture)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _run(spec, cuts, resident, monkeypatch, provider=None):
    from paper_2104_11385_b200.workload import Simulation
    if resident:
        monkeypatch.delenv("LBX_NO_RESIDENT", raising=False)
    else:
        monkeypatch.setenv("LBX_NO_RESIDENT", "1")
    sim = Simulation(spec.scenario, spec.policy, provider or spec.build_provider(),
                     device="cuda:0", record_counts=True, record_clock=True)
    for a, b in zip(cuts[:-1], cuts[1:]):
        sim.run(a, b)
    used = sim.resident_runs
    res = sim.result()
    sim.close()
    return res, used


def _same(a, b):
    assert np.array_equal(a.cost_trace, b.cost_trace)
    assert np.array_equal(a.count_trace, b.count_trace)
    for k in ("efficiency_before", "efficiency_after", "adopted", "walltime",
              "max_rank_particles"):
        assert [getattr(m, k) for m in a.metrics] == [getattr(m, k) for m in b.metrics], k
    assert [[s, o.tolist()] for s, o in a.adoption_snapshots] == \
        [[s, o.tolist()] for s, o in b.adoption_snapshots]
    ap, av = a.final_state.to_numpy()
    bp, bv = b.final_state.to_numpy()
    assert np.array_equal(ap, bp) and np.array_equal(av, bv)


@pytest.mark.parametrize("name", ["mini", "mini_measured", "c1", "small", "leaky",
                                  "default_short"])
def test_resident_matches_per_step_path(runs, name, monkeypatch):  # noqa: F811
    spec = spec_for(runs, name)
    T = spec.scenario.total_steps
    k = spec.scenario.kick.step
    cuts = sorted({0, 3, max(k - 1, 4), min(k + 1, T - 1), k + 7 if k + 7 < T else T - 2, T})
    r, used = _run(spec, cuts, True, monkeypatch)
    p, none = _run(spec, cuts, False, monkeypatch)
    assert none == 0
    assert used == sum(b - a >= 2 for a, b in zip(cuts[:-1], cuts[1:])), (used, cuts)
    _same(r, p)
    assert sha(r.cost_trace) == runs[name]["cost_trace_sha"]
    fp, fv = r.final_state.to_numpy()
    assert sha(fp) == runs[name]["final_pos_sha"] and sha(fv) == runs[name]["final_vel_sha"]


@pytest.mark.parametrize("name", ["mini", "default_short"])
def test_resident_gpuclock_counts_and_tally(runs, name, monkeypatch):  # noqa: F811
    """GpuClock on the resident kernel: per-box counts (and so the heuristic
    columns / final state) equal the per-step path's; every occupied box
    gets a positive clock tally and the tally ranks boxes like their counts."""
    from paper_2104_11385_b200 import scenarios as S
    spec = S.apply_overrides(spec_for(runs, name), cost="gpuclock")
    T = spec.scenario.total_steps
    r, used = _run(spec, [0, T // 3, T], True, monkeypatch)
    p, _ = _run(spec, [0, T // 3, T], False, monkeypatch)
    assert used == 2
    assert np.array_equal(r.count_trace, p.count_trace)
    rp, rv = r.final_state.to_numpy()
    pp, pv = p.final_state.to_numpy()
    assert np.array_equal(rp, pp) and np.array_equal(rv, pv)
    ct = r.clock_trace
    assert ct is not None
    occ = r.count_trace > 0
    assert (ct[occ] > 0).all() and (ct[~occ] == 0).all()
