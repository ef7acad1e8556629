"""CPU tests of libLBX's host side: symbol exports and the bit-exact
balancer / PCG64 restatement against reference fixtures (no GPU needed)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import lbsim_oracle as O

ROOT = Path(__file__).resolve().parent.parent
G = ROOT / "tests" / "golden"


@pytest.fixture(scope="module")
def L():
    from paper_2104_11385_b200 import _lib
    return _lib


def test_library_exports_every_header_symbol(L):
    header = (ROOT / "include" / "lbx.h").read_text()
    names = set(re.findall(r"^\s*(?:int|double|const char\*)\s+(lbx_\w+)\(", header, re.M))
    assert names, "no declarations parsed"
    assert names == set(L.SIGNATURES), names ^ set(L.SIGNATURES)
    lib = C.CDLL(str(L.LIB_PATH))
    for n in names:
        assert hasattr(lib, n), n


def _ks(L, c, R, cap):
    c = np.ascontiguousarray(c, dtype=np.float64)
    out = np.empty(c.size, dtype=np.int64)
    L.check(L.lib.lbx_knapsack(L.ptr(c), c.size, R, cap, L.ptr(out)))
    return out


def _sfc(L, c, curve, R):
    c = np.ascontiguousarray(c, dtype=np.float64)
    curve = np.ascontiguousarray(curve, dtype=np.int64)
    out = np.empty(c.size, dtype=np.int64)
    L.check(L.lib.lbx_sfc(L.ptr(c), L.ptr(curve), c.size, R, L.ptr(out)))
    return out


def _eff(L, c, owner, R):
    c = np.ascontiguousarray(c, dtype=np.float64)
    owner = np.ascontiguousarray(owner, dtype=np.int64)
    e, d = C.c_double(), C.c_int32()
    L.check(L.lib.lbx_efficiency(L.ptr(c), L.ptr(owner), c.size, R, C.byref(e), C.byref(d)))
    return e.value, bool(d.value)


def _morton(L, nbz, nbx):
    out = np.empty(nbz * nbx, dtype=np.int64)
    L.check(L.lib.lbx_morton_order(nbz, nbx, L.ptr(out)))
    return out


def test_balancer_matches_reference_fixture(L):
    f = np.load(G / "balancer.npz")
    for i, (nbz, nbx, R, cap, e_ks, e_sf) in enumerate(f["meta"]):
        R = int(R)
        c = f[f"c{i}"]
        curve = _morton(L, int(nbz), int(nbx))
        assert np.array_equal(curve, f[f"m{i}"])
        if f[f"k{i}"][0] >= 0:
            ks = _ks(L, c, R, cap)
            assert np.array_equal(ks, f[f"k{i}"]), i
            assert _eff(L, c, ks, R)[0] == e_ks
        else:
            with pytest.raises(ValueError, match="cap"):
                _ks(L, c, R, cap)
        sf = _sfc(L, c, curve, R)
        assert np.array_equal(sf, f[f"s{i}"]), i
        assert _eff(L, c, sf, R)[0] == e_sf
    for R in (8, 24):
        assert np.array_equal(_ks(L, f["big_c"], R, 1.5), f[f"big_k{R}"])
        assert np.array_equal(_sfc(L, f["big_c"], f["big_curve"], R), f[f"big_s{R}"])


def test_random_balancer_vs_oracle(L):
    rng = np.random.default_rng(123)
    for _ in range(300):
        n = int(rng.integers(1, 200))
        R = int(rng.integers(1, 12))
        c = rng.random(n) * 10 ** rng.uniform(-2, 5)
        if rng.random() < 0.3:
            c = np.round(c)
        try:
            want = O.knapsack_assign(c, R, 1.5)
        except ValueError:
            continue
        assert np.array_equal(_ks(L, c, R, 1.5), want)
        curve = rng.permutation(n)
        assert np.array_equal(_sfc(L, c, curve, R), O.sfc_assign(c, curve, R))
        own = rng.integers(0, R, n)
        assert _eff(L, c, own, R) == O.efficiency_flagged(c, own, R)


def test_pairwise_sum_matches_numpy(L):
    rng = np.random.default_rng(1)
    for n in list(range(0, 300)) + [1000, 4099, 8192, 10001, 65537]:
        a = rng.random(n) * 10 ** rng.uniform(-3, 3, n)
        assert L.lib.lbx_pairwise_sum(L.ptr(a), n) == (a.sum() if n else 0.0)


def test_measured_cost_matches_reference_fixture(L):
    f = np.load(G / "measured.npz")
    amps = {"7_0_900": 0.05, "11_123_225": 0.05, "13_599_900": 0.2, "0_5_17": 0.5,
            f"{2**40+3}_{2**33}_64": 0.05}
    for key, amp in amps.items():
        seed, step, n = (int(x) for x in key.split("_"))
        work = np.linspace(1.0, 1000.0, n)
        out = np.empty(n)
        L.check(L.lib.lbx_measured_cost(L.ptr(work), n, amp, seed, step, L.ptr(out)))
        assert np.array_equal(out, f[key]), key


def test_slab_and_morton_vs_oracle(L):
    for nb in (1, 7, 16, 225, 900, 1000):
        for R in (1, 3, 8, 24, 37):
            out = np.empty(nb, dtype=np.int64)
            L.check(L.lib.lbx_slab_mapping(nb, R, L.ptr(out)))
            assert np.array_equal(out, O.slab_mapping(nb, R)), (nb, R)
    for nbz, nbx in ((1, 1), (2, 2), (30, 30), (3, 17), (16, 5)):
        assert np.array_equal(_morton(L, nbz, nbx), O.morton_order(nbz, nbx))


def test_contract_errors(L):
    with pytest.raises(ValueError, match="permutation"):
        _sfc(L, [1.0, 2.0], [0, 0], 2)
    with pytest.raises(ValueError, match="empty"):
        _sfc(L, np.empty(0), np.empty(0, np.int64), 2)
    with pytest.raises(ValueError, match="n_ranks"):
        _ks(L, [1.0], 0, 1.5)
    with pytest.raises(ValueError, match="owner"):
        _eff(L, [1.0, 2.0], [0, 5], 2)


def test_morton_3d_vs_oracle(L):
    for g in ((1, 1, 1), (2, 2, 2), (8, 8, 4), (3, 5, 2)):
        out = np.empty(g[0] * g[1] * g[2], dtype=np.int64)
        L.check(L.lib.lbx_morton_order_3d(*g, L.ptr(out)))
        assert np.array_equal(out, O.morton_order_3d(g)), g


def test_migration_aware_gate(L):
    """B200 extension: a huge migration price blocks the
    adoption the reference gate would make; zero restores the reference."""
    import ctypes as C

    from paper_2104_11385_b200.balancer import BalancePolicy
    from paper_2104_11385_b200.cost import make_provider
    from paper_2104_11385_b200.scenarios import load_spec
    from paper_2104_11385_b200.workload import sim_config
    sc = load_spec("mini").scenario
    counts = np.zeros(225, dtype=np.int64)
    counts[:20] = 1000            # all load on rank 0 of a slab mapping
    owner = O.slab_mapping(225, 8)
    res = {}
    for ratio in (0.0, 1e9):
        conf = sim_config(sc, BalancePolicy(migration_ratio=ratio), make_provider("heuristic"))
        h = C.c_void_p()
        L.check(L.lib.lbx_lb_create(C.byref(h), C.byref(conf), L.ptr(owner)))
        T, nb = sc.total_steps, 225
        arrs = {k: np.zeros(T) for k in ("eb", "ea", "cm", "co", "g", "r", "w")}
        u8 = {k: np.zeros(T, dtype=np.uint8) for k in ("ad", "at", "oom")}
        i64 = {k: np.zeros(T, dtype=np.int64) for k in ("mrp", "na", "as")}
        trace = np.zeros((T, nb))
        own_out = owner.copy()
        so = L.SimOutputs(L.ptr(arrs["eb"]), L.ptr(arrs["ea"]), L.ptr(u8["ad"]), L.ptr(u8["at"]),
                          L.ptr(arrs["cm"]), L.ptr(arrs["co"]), L.ptr(arrs["g"]), L.ptr(arrs["r"]),
                          L.ptr(arrs["w"]), L.ptr(i64["mrp"]), L.ptr(u8["oom"]), L.ptr(i64["na"]),
                          L.ptr(trace), None, None, L.ptr(own_out), L.ptr(i64["as"]), None, None,
                          0, 0, 0)
        ad, halt = C.c_int32(), C.c_int32()
        L.check(L.lib.lbx_lb_step(h, 0, L.ptr(counts), None, int(counts.sum()), C.byref(so),
                                  C.byref(ad), C.byref(halt)))
        L.lib.lbx_lb_destroy(h)
        res[ratio] = ad.value
    assert res[0.0] == 1 and res[1e9] == 0


def _native_adopt(L, sc, owner, counts, ratio):
    import ctypes as C

    from paper_2104_11385_b200.balancer import BalancePolicy
    from paper_2104_11385_b200.cost import make_provider
    from paper_2104_11385_b200.workload import sim_config
    conf = sim_config(sc, BalancePolicy(migration_ratio=ratio), make_provider("heuristic"))
    h = C.c_void_p()
    L.check(L.lib.lbx_lb_create(C.byref(h), C.byref(conf), L.ptr(owner)))
    T, nb = sc.total_steps, owner.size
    arrs = [np.zeros(T) for _ in range(7)]
    u8 = [np.zeros(T, dtype=np.uint8) for _ in range(3)]
    i64 = [np.zeros(T, dtype=np.int64) for _ in range(3)]
    trace = np.zeros((T, nb))
    own_out = owner.copy()
    so = L.SimOutputs(*(L.ptr(a) for a in arrs[:2]), L.ptr(u8[0]), L.ptr(u8[1]),
                      *(L.ptr(a) for a in arrs[2:7]), L.ptr(i64[0]), L.ptr(u8[2]),
                      L.ptr(i64[1]), L.ptr(trace), None, None, L.ptr(own_out), L.ptr(i64[2]),
                      None, None, 0, 0, 0)
    ad, halt = C.c_int32(), C.c_int32()
    L.check(L.lib.lbx_lb_step(h, 0, L.ptr(counts), None, int(counts.sum()), C.byref(so),
                              C.byref(ad), C.byref(halt)))
    L.lib.lbx_lb_destroy(h)
    return bool(ad.value)


def test_python_gate_applies_migration_ratio_like_native(L):
    """the Python attempt_rebalance applies the same migration-
    aware check as the native lb_step (same decision on both sides of the
    break-even ratio), and refuses to run it without counts."""
    from paper_2104_11385_b200.balancer import BalancePolicy, attempt_rebalance
    from paper_2104_11385_b200.cost import CostVector
    from paper_2104_11385_b200.decomposition import DistributionMapping
    from paper_2104_11385_b200.scenarios import load_spec
    sc = load_spec("mini").scenario
    rng = np.random.default_rng(3)
    for trial in range(6):
        counts = np.zeros(225, dtype=np.int64)
        k = int(rng.integers(5, 60))
        counts[:k] = rng.integers(100, 5000, size=k)
        owner = O.slab_mapping(225, 8)
        cv = CostVector(values=O.heuristic_cost(counts, np.full(225, sc.box_size ** 2),
                                                0.75, 0.25), step=0)
        dm = DistributionMapping(owner=owner, n_ranks=8)
        with pytest.raises(ValueError, match="counts"):
            attempt_rebalance(cv, dm, BalancePolicy(migration_ratio=1.0), 0)
        for ratio in (0.0, 0.5, 2.0, 8.0, 30.0, 1e3, 1e9):
            py = attempt_rebalance(cv, dm, BalancePolicy(migration_ratio=ratio), 0,
                                   counts=counts).adopted
            assert py == _native_adopt(L, sc, owner, counts, ratio), (trial, ratio)


def test_integration_md_ctypes_binding():
    """The raw ctypes binding INTEGRATION.md shows a reference maintainer
    (no package import, plain CDLL + argtypes) gives the oracle's owners."""
    import ctypes as C
    from pathlib import Path

    import numpy as np

    from oracle import lbsim_oracle as O
    so = Path(__file__).resolve().parent.parent / "paper_2104_11385_b200" / "libLBX.so"
    lib = C.CDLL(str(so))
    lib.lbx_knapsack.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_void_p]
    lib.lbx_last_error.restype = C.c_char_p
    rng = np.random.default_rng(7)
    v = np.ascontiguousarray(rng.uniform(0, 100, 300))
    owner = np.empty(v.size, dtype=np.int64)
    assert lib.lbx_knapsack(v.ctypes.data, v.size, 8, 1.5, owner.ctypes.data) == 0
    assert np.array_equal(owner, np.asarray(O.knapsack_assign(v, 8, 1.5)))
    bad = np.ascontiguousarray(np.ones(10))
    assert lib.lbx_knapsack(bad.ctypes.data, bad.size, 8, 0.5, owner.ctypes.data) != 0
    assert b"cap" in lib.lbx_last_error()
