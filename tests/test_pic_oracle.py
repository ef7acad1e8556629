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


def _div_j(j):
    d = np.zeros_like(j["Jz"])
    d[1:, :] += j["Jz"][1:, :] - j["Jz"][:-1, :]
    d[0, :] += j["Jz"][0, :]
    d[:, 1:] += j["Jx"][:, 1:] - j["Jx"][:, :-1]
    d[:, 0] += j["Jx"][:, 0]
    return d


def test_shapes_partition_unity():
    rng = np.random.default_rng(4)
    pos = rng.uniform(3, 20, 5000)
    for order in PO.SHAPE_ORDERS:
        b = PO.shape_base(pos, order)
        w = PO.window_weights(pos, b, order, order + 1)
        assert np.max(np.abs(w.sum(axis=1) - 1.0)) < 1e-14, order
        assert (w >= 0).all()
        # the window is exactly the support: one node further has zero weight
        assert np.all(PO.window_weights(pos, b - 1, order, 1) == 0.0)


def test_esirkepov_continuity_all_orders():
    """drho/dt + div J = 0 to rounding for shape orders 1-3 (the paper's
    order-3 deposition), for moves up to 0.9 cell per axis."""
    rng = np.random.default_rng(5)
    n, nz, nx, pad, qw, dt = 3000, 24, 24, 4, -0.05, 0.5
    shape = (nz + 2 * pad, nx + 2 * pad)
    for order in PO.SHAPE_ORDERS:
        z0, x0 = rng.uniform(6, 18, n), rng.uniform(6, 18, n)
        z1, x1 = z0 + rng.uniform(-0.9, 0.9, n), x0 + rng.uniform(-0.9, 0.9, n)
        j = PO.esirkepov_current(z0, x0, z1, x1, rng.normal(0, 0.1, n), qw, dt, order, shape,
                                 pad)
        r0 = PO.deposit_rho(z0, x0, qw, order, shape, pad)
        r1 = PO.deposit_rho(z1, x1, qw, order, shape, pad)
        res = (r1 - r0) / dt + _div_j(j)
        assert np.abs(res).max() < 1e-12 * np.abs(r1).max() * n ** 0.5, order
        assert np.abs(j["Jz"]).max() > 0 and np.abs(j["Jx"]).max() > 0


def test_esirkepov_order1_jy_matches_average_shape():
    """Jy of the charge-conserving scheme at zero displacement is q w vy S0 S0."""
    rng = np.random.default_rng(6)
    n, pad = 500, 3
    z, x = rng.uniform(5, 10, n), rng.uniform(5, 10, n)
    vy = rng.normal(0, 0.2, n)
    for order in PO.SHAPE_ORDERS:
        j = PO.esirkepov_current(z, x, z, x, vy, -0.05, 0.5, order, (16 + 2 * pad,) * 2, pad)
        rho_v = np.zeros_like(j["Jy"])
        for i in range(n):
            rho_v += PO.deposit_rho(z[i:i + 1], x[i:i + 1], -0.05 * vy[i], order,
                                    rho_v.shape, pad)
        assert np.max(np.abs(j["Jy"] - rho_v)) < 1e-13
        assert np.abs(j["Jz"]).max() == 0 and np.abs(j["Jx"]).max() == 0


def test_esirkepov_step_energy_is_conserved():
    """Whole PIC steps (shaped gather, Boris, Esirkepov deposit, Yee) of a
    warm plasma: total (field + kinetic) energy stays within 3 % (order 1)
    and 1 % (order 3) over 40 steps; the field energy actually grows from
    zero, so the check is not vacuous."""
    rng = np.random.default_rng(1)
    nz = nx = 32
    n, qm, qw, dt = 20000, -1.0, -0.02, 0.5
    for order, tol in ((1, 0.03), (3, 0.01)):
        p = {"z": rng.uniform(8, 24, n), "x": rng.uniform(8, 24, n),
             "uz": rng.normal(0, 0.1, n), "ux": rng.normal(0, 0.1, n),
             "uy": rng.normal(0, 0.1, n)}
        f = PO.new_fields(nz, nx)
        tot, fe = [], []
        for _ in range(40):
            PO.particle_step_esirkepov(f, p, nz, nx, qm, qw, dt, order)
            PO.field_step(f, nz, nx, dt)
            fe.append(PO.field_energy(f))
            tot.append(fe[-1] + PO.kinetic_energy(p, qw / qm))
        tot = np.array(tot)
        assert (tot.max() - tot.min()) / tot.mean() < tol, order
        assert max(fe) > 0.01 * tot.mean()
