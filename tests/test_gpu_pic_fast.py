"""Tolerance mode of the PIC step (LBX_PIC_FAST, pic_fast_kernel) against the
fp64 numpy oracle (oracle/pic_oracle.py).  Parity unpinned by the reference
(no PIC there); the oracle is the builder's restatement.  north_star allows
fields and particle state to agree "within a stated fp32/fp64 tolerance";
the tolerances below follow from the mode's arithmetic:

* momenta: the Boris update is computed in float32 as the INCREMENT du and
  added to the fp64 momenta, so |du_gpu - du_oracle| <~ few ulp32 of |du| +
  the FMA-lerp gather difference (ulp32 of the field)  ->  U_TOL relative to
  max |u|;
* positions: x += float32(dt u / gamma): <~ ulp32 of the per-step move,
  accumulated over the steps  ->  X_TOL cells;
* current: node values rounded on the run's float32 moment sums instead of
  per particle: <~ a few ulp32 of the run sum per node  ->  J_TOL relative
  to max |J|;
* fields: E, B inherit the current's and the gathers' relative error ->
  F_TOL relative to each component's max.
Per-box particle counts (integers) must be exact."""
import numpy as np
import pytest

from oracle import lbsim_oracle as LO
from oracle import pic_oracle as PO
from tests.test_gpu_pic import setup

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

U_TOL = 2e-6      # |du| error / max |u|
X_TOL = 1e-6      # cells
J_TOL = 2e-5      # / max |J| per component
F_TOL = 2e-4      # / max |F| per component


def run_fast(pos, u, nz, nx, steps, field_solve=True, qm=-1.0, qw=-0.05, dt=0.5, M=16,
             gather=None, stable=True, fields=None, tiled=False):
    from paper_2104_11385_b200 import device, pic
    ctx = device.Context(capacity=pos.shape[0])
    st = pic.PicState.create(pos, u, nz, nx)
    if tiled:   # tile-major order + ranges (the particle order then differs from the oracle's)
        pic.pic_sort(ctx, st, tiled=True)
    f = PO.new_fields(nz, nx)
    if fields is not None:        # seed nonzero fields so the push sees E and B
        for k, v in fields.items():
            f[k][:] = v
        for k, t in st.fields.items():
            t.copy_(torch.from_numpy(f[k]).to(t.device))
    p = {"z": pos[:, 0].copy(), "x": pos[:, 1].copy(), "uz": u[:, 0].copy(),
         "ux": u[:, 1].copy(), "uy": u[:, 2].copy()}
    outs = []
    for _ in range(steps):
        out = pic.pic_step(ctx, st, M, qm, qw, dt, field_solve=field_solve, clock=True,
                           gather=gather, stable=stable, fast=True, tiled=tiled)
        PO.particle_step(f, p, nz, nx, qm, qw, dt)
        fj = {k: f[k].copy() for k in ("Jx", "Jy", "Jz")}
        c = LO.bin_particles(np.column_stack([p["z"], p["x"]]), float(M), nz // M, nx // M)
        if field_solve:
            PO.field_step(f, nz, nx, dt)
        outs.append((out, fj, c))
    return st, f, p, outs


def seeded_fields(nz, nx, seed, amp=0.05):
    rng = np.random.default_rng(seed)
    out = {}
    for k in PO.OFFSETS:
        a = np.zeros((nz + 2, nx + 2), dtype=np.float32)
        a[1:-1, 1:-1] = rng.normal(0, amp, size=(nz, nx)).astype(np.float32)
        out[k] = a
    return out


def rel_err(a, b):
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


@pytest.mark.parametrize("gather", ["quad", "direct"])
@pytest.mark.parametrize("clustered", [True, False])
def test_fast_mode_within_tolerance(clustered, gather):
    nz, nx = 64, 96
    pos, u = setup(40_000, nz, nx, seed=2, clustered=clustered)
    st, f, p, outs = run_fast(pos, u, nz, nx, steps=6, gather=gather,
                              fields=seeded_fields(nz, nx, 5))
    for out, _, c in outs:
        assert np.array_equal(out["counts"], c)
    g = st.particles()
    assert g["z"].shape == p["z"].shape
    umax = max(np.max(np.abs(p[k])) for k in ("uz", "ux", "uy"))
    for k in ("uz", "ux", "uy"):
        e = np.max(np.abs(g[k] - p[k])) / umax
        assert e <= U_TOL, (k, e)
    for k in ("z", "x"):
        e = np.max(np.abs(g[k] - p[k]))
        assert e <= X_TOL, (k, e)
    fa = st.field_arrays()
    for k in PO.OFFSETS:
        e = rel_err(fa[k], f[k])
        assert e <= F_TOL, (k, e)


def test_fast_mode_first_step_current():
    """The current of one step (no field solve) within J_TOL of the oracle's,
    for a dense clustered plasma (long same-cell runs: the moment sums) and
    a scattered one (runs of one: per-particle rounding)."""
    for clustered in (True, False):
        nz = nx = 64
        pos, u = setup(60_000, nz, nx, seed=1, clustered=clustered)
        st, f, p, outs = run_fast(pos, u, nz, nx, steps=1, field_solve=False,
                                  fields=seeded_fields(nz, nx, 3))
        fa = st.field_arrays()
        for k in ("Jx", "Jy", "Jz"):
            ref = outs[0][1][k]
            assert np.abs(ref).max() > 0
            e = rel_err(fa[k], ref)
            assert e <= J_TOL, (clustered, k, e)


def test_fast_mode_absorption():
    pos, u = setup(30_000, 32, 32, seed=3, speed=2.0, clustered=False)
    st, f, p, outs = run_fast(pos, u, 32, 32, steps=4, field_solve=False)
    assert st.n == p["z"].size < 30_000
    g = st.particles()
    for k in ("z", "x"):
        assert np.max(np.abs(g[k] - p[k])) <= X_TOL


def test_fast_mode_hole_filling_keeps_the_multiset():
    """Without stable order, absorbed slots are filled from the tail: the
    particle multiset still matches the oracle's within tolerance."""
    pos, u = setup(30_000, 32, 32, seed=4, speed=2.0, clustered=False)
    st, f, p, outs = run_fast(pos, u, 32, 32, steps=3, field_solve=False, stable=False)
    assert st.n == p["z"].size
    g = st.particles()
    # per-column sorted values: a multiset check that near-ties (two
    # particles closer than the tolerance) cannot break
    umax = max(np.max(np.abs(p[k])) for k in ("uz", "ux", "uy"))
    for k in ("z", "x"):
        assert np.max(np.abs(np.sort(g[k]) - np.sort(p[k]))) <= X_TOL
    for k in ("uz", "ux", "uy"):
        assert np.max(np.abs(np.sort(g[k]) - np.sort(p[k]))) <= U_TOL * umax


@pytest.mark.parametrize("clustered", [True, False])
def test_fast_tiled_within_tolerance(clustered):
    """Tolerance mode on the tiled path (LBX_PIC_FAST | LBX_PIC_TILED, the
    sparse-plasma kernel): after a tile-major sort and 6 steps with the field
    solve, the particle multiset, the fields and the per-box counts agree
    with the fp64 oracle at the same tolerances."""
    nz, nx = 64, 96
    pos, u = setup(40_000, nz, nx, seed=7, clustered=clustered)
    st, f, p, outs = run_fast(pos, u, nz, nx, steps=6, stable=False, tiled=True,
                              fields=seeded_fields(nz, nx, 9))
    for out, _, c in outs:
        assert np.array_equal(out["counts"], c)
    g = st.particles()
    assert g["z"].shape == p["z"].shape
    umax = max(np.max(np.abs(p[k])) for k in ("uz", "ux", "uy"))
    for k in ("z", "x"):
        assert np.max(np.abs(np.sort(g[k]) - np.sort(p[k]))) <= X_TOL, k
    for k in ("uz", "ux", "uy"):
        assert np.max(np.abs(np.sort(g[k]) - np.sort(p[k]))) <= U_TOL * umax, k
    fa = st.field_arrays()
    for k in PO.OFFSETS:
        e = rel_err(fa[k], f[k])
        assert e <= F_TOL, (k, e)


def test_pipelined_kernel_on_a_large_sparse_grid():
    """Regression (round 2): in the last, partial chunk of pic_pipe_kernel the
    slots past the end of the array read the shared quad window at an index
    computed from cell 0 -- outside the CTA's shared memory when the window
    sits at large cell indices (an illegal-address fault on a 2048^2 grid).
    A uniform 2048^2 x 8 ppc plasma (33.5 M particles) through the pipelined
    kernel (quad gather forced) in the exact mode: per-box counts and the
    particle count agree with the exact tiled path on the same input."""
    from paper_2104_11385_b200 import device, pic
    nz = nx = 2048
    rng = np.random.default_rng(42)
    cell = np.repeat(np.arange(nz * nx, dtype=np.int64), 8)
    off = rng.random((cell.size, 2))
    pos = np.column_stack([(cell // nx) + off[:, 0], (cell % nx) + off[:, 1]])
    u = rng.normal(0.0, 0.05, size=(cell.size, 3))
    del cell, off
    outs = {}
    for mode in ("pipe", "tiled"):
        ctx = device.Context(capacity=pos.shape[0])
        st = pic.PicState.create(pos, u, nz, nx)
        pic.pic_sort(ctx, st, tiled=mode == "tiled")
        res = []
        for _ in range(2):
            if mode == "pipe":
                out = pic.pic_step(ctx, st, 128, -1.0, -1e-4, 0.5, gather="quad")
            else:
                out = pic.pic_step(ctx, st, 128, -1.0, -1e-4, 0.5, tiled=True)
            res.append((out["n"], out["counts"].copy()))
        outs[mode] = res
        del st, ctx
        torch.cuda.empty_cache()
    for (na, ca), (nb, cb) in zip(outs["pipe"], outs["tiled"]):
        assert na == nb < pos.shape[0]
        assert np.array_equal(ca, cb)
