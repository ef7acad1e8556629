"""2D3V PIC step (gather + Boris + deposit + Yee) vs the fp64/fp32 numpy
oracle.  Parity unpinned by the reference (no PIC there); tolerances:
  * step 1 from zero fields: particles bit-exact (no field contribution);
  * currents / fields: max |GPU - oracle| <= 1e-5 * max|oracle| + 1e-7
    (float32 atomics sum in a different order);
  * particles after N steps: |dz|, |dx| <= 1e-6 cells, |du| <= 1e-6;
  * per-box counts: exact while no particle sits within 1e-6 of a box edge.
"""
import numpy as np
import pytest

from oracle import lbsim_oracle as LO
from oracle import pic_oracle as PO

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def setup(n, nz, nx, seed, speed=0.3, clustered=True):
    rng = np.random.default_rng(seed)
    if clustered:   # blob-like, spatially sorted (exercises staged patches)
        c = np.array([nz / 2, nx / 2])
        r = rng.random(n) ** 0.5 * min(nz, nx) * 0.3
        a = rng.random(n) * 2 * np.pi
        pos = np.column_stack([c[0] + r * np.cos(a), c[1] + r * np.sin(a)])
        pos = pos[np.lexsort((pos[:, 1], np.floor(pos[:, 0])))]
    else:           # scattered: exercises the global fallback path
        pos = rng.uniform(0, [nz, nx], size=(n, 2))
    u = rng.normal(0, speed, size=(n, 3))
    return pos, u


def run_both(pos, u, nz, nx, steps, field_solve=True, qm=-1.0, qw=-0.05, dt=0.5, M=16):
    from paper_2104_11385_b200 import device, pic
    ctx = device.Context(capacity=pos.shape[0])
    st = pic.PicState.create(pos, u, nz, nx)
    f = PO.new_fields(nz, nx)
    p = {"z": pos[:, 0].copy(), "x": pos[:, 1].copy(), "uz": u[:, 0].copy(),
         "ux": u[:, 1].copy(), "uy": u[:, 2].copy()}
    outs = []
    for _ in range(steps):
        out = pic.pic_step(ctx, st, M, qm, qw, dt, field_solve=field_solve, clock=True)
        PO.particle_step(f, p, nz, nx, qm, qw, dt)
        fj = {k: f[k].copy() for k in ("Jx", "Jy", "Jz")}
        if field_solve:
            PO.field_step(f, nz, nx, dt)
        outs.append((out, fj))
    return st, f, p, outs


def close(a, b, rel=1e-5, abs_=1e-7):
    return np.max(np.abs(a - b)) <= rel * max(np.max(np.abs(b)), 1e-30) + abs_


def test_first_step_particles_exact_and_currents_close():
    pos, u = setup(60_000, 64, 64, seed=1)
    st, f, p, outs = run_both(pos, u, 64, 64, steps=1, field_solve=False)
    g = st.particles()
    for k in ("z", "x", "uz", "ux", "uy"):
        assert np.array_equal(g[k], p[k]), k
    fa = st.field_arrays()
    for k in ("Jx", "Jy", "Jz"):
        assert close(fa[k], outs[0][1][k]), k
    c = LO.bin_particles(np.column_stack([p["z"], p["x"]]), 16.0, 4, 4)
    assert np.array_equal(outs[0][0]["counts"], c)
    assert ((outs[0][0]["clock"] > 0) == (c > 0)).all()


@pytest.mark.parametrize("clustered", [True, False])
def test_multi_step_with_field_solve(clustered):
    pos, u = setup(40_000, 64, 96, seed=2, clustered=clustered)
    st, f, p, outs = run_both(pos, u, 64, 96, steps=6, field_solve=True)
    g = st.particles()
    assert g["z"].shape == p["z"].shape
    for k in ("z", "x"):
        assert np.max(np.abs(g[k] - p[k])) <= 1e-6, k
    for k in ("uz", "ux", "uy"):
        assert np.max(np.abs(g[k] - p[k])) <= 1e-6, k
    fa = st.field_arrays()
    for k in PO.OFFSETS:
        assert close(fa[k], f[k], rel=1e-4, abs_=1e-6), k
    assert np.max(np.abs(fa["Ey"])) > 0          # fields actually evolved


def test_absorption_and_compaction_keep_order():
    pos, u = setup(30_000, 32, 32, seed=3, speed=2.0, clustered=False)
    st, f, p, outs = run_both(pos, u, 32, 32, steps=4, field_solve=False)
    g = st.particles()
    assert st.n == p["z"].size < 30_000
    assert np.max(np.abs(g["z"] - p["z"])) <= 1e-6
