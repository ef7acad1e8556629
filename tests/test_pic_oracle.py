"""CPU self-checks of the PIC oracle (oracle/pic_oracle.py).  The reference
has no PIC, so the oracle is pinned by physics identities instead of golden
vectors: Boris rotation preserves |u| in a pure magnetic field, the
half-staggered stencil equals the floor(z - 1/2) stencil, the fixed-point
deposit conserves the particle current up to rounding and is additive over
particle subsets (what makes the multi-GPU reduction exact), and the Yee
update leaves a uniform field (zero curl) unchanged."""
import numpy as np

from oracle import pic_oracle as PO


def test_boris_pure_b_rotation_preserves_speed():
    rng = np.random.default_rng(0)
    n = 1000
    u = rng.normal(0, 0.5, size=(3, n))
    E = {k: np.zeros(n) for k in PO.E_COMPS}
    B = {k: rng.normal(0, 0.3, n) for k in PO.B_COMPS}
    uz, ux, uy = PO.boris(u[0], u[1], u[2], E, B, -1.0, 0.5)
    before = u[0] ** 2 + u[1] ** 2 + u[2] ** 2
    after = uz ** 2 + ux ** 2 + uy ** 2
    assert np.max(np.abs(after - before) / before) < 1e-13
    assert not np.allclose(uz, u[0])       # it did rotate


def test_half_stagger_stencil_matches_floor_of_shifted_position():
    rng = np.random.default_rng(1)
    z = rng.uniform(1.0, 900.0, 100_000)
    i, f = PO._axis(z, 0.5)
    zc = z - 0.5
    assert np.array_equal(i, np.floor(zc).astype(np.int64))
    ref = (zc - np.floor(zc)).astype(np.float32)
    assert np.max(np.abs(f - ref)) <= np.finfo(np.float32).eps
    i0, f0 = PO._axis(z, 0.0)
    assert np.array_equal(i0, np.floor(z).astype(np.int64))


def test_deposit_conserves_current_and_is_additive():
    rng = np.random.default_rng(2)
    n, nz, nx = 5000, 16, 24
    p = {"z": rng.uniform(0, nz, n), "x": rng.uniform(0, nx, n),
         "uz": rng.normal(0, 0.2, n), "ux": rng.normal(0, 0.2, n), "uy": rng.normal(0, 0.2, n)}
    ig = 1.0 / np.sqrt(1.0 + p["uz"] ** 2 + p["ux"] ** 2 + p["uy"] ** 2)
    qw = -0.05
    shape = (nz + 2, nx + 2)
    accs = PO.current_accs(p, ig, qw, shape)
    sc = PO.current_scale(qw)
    for comp, u in (("Jx", p["ux"]), ("Jy", p["uy"]), ("Jz", p["uz"])):
        v = (qw * u * ig).astype(np.float32).astype(np.float64) * sc
        assert abs(accs[comp].sum() - v.sum()) <= 2.0 * n       # <= 4 x 0.5 per particle
    half = {k: a[: n // 2] for k, a in p.items()}
    rest = {k: a[n // 2:] for k, a in p.items()}
    a1 = PO.current_accs(half, ig[: n // 2], qw, shape)
    a2 = PO.current_accs(rest, ig[n // 2:], qw, shape)
    for comp in accs:
        assert np.array_equal(a1[comp] + a2[comp], accs[comp])


def test_yee_uniform_field_is_stationary():
    nz, nx = 12, 10
    f = PO.new_fields(nz, nx)
    s = (slice(1, nz + 1), slice(1, nx + 1))
    f["Ey"][s] = 0.25
    before = {k: v.copy() for k, v in f.items()}
    PO.field_step(f, nz, nx, 0.5)
    interior = (slice(2, nz), slice(2, nx))     # away from the conducting walls
    for k in PO.OFFSETS:
        assert np.array_equal(f[k][interior], before[k][interior]), k


def test_particle_step_moves_and_absorbs():
    rng = np.random.default_rng(3)
    n, nz, nx = 2000, 8, 8
    p = {"z": rng.uniform(0, nz, n), "x": rng.uniform(0, nx, n),
         "uz": rng.normal(0, 2.0, n), "ux": rng.normal(0, 2.0, n), "uy": np.zeros(n)}
    f = PO.new_fields(nz, nx)
    keep = PO.particle_step(f, p, nz, nx, -1.0, -0.01, 0.5)
    assert 0 < keep.sum() < n and p["z"].size == keep.sum()
    assert ((p["z"] >= 0) & (p["z"] < nz) & (p["x"] >= 0) & (p["x"] < nx)).all()
    assert np.abs(f["Jz"]).max() > 0
