"""CPU oracle for the 2D3V PIC step -- TEST INFRASTRUCTURE ONLY.

PARITY UNPINNED: the reference (lbsim) has no particle-in-cell physics; the
paper's WarpX step is only described.  This
module is the builder's own restatement of the algorithm the CUDA kernels
implement (paper_2104_11385_b200/csrc/lbx_pic.cu), used as the numerical
checker at a stated tolerance.  Only tests/ may import it.

Algorithm (normalised units: c = 1, cell size 1, charge/mass q/m per species,
macro weight w):
  fields  Yee grid, 2D in (z, x), y invariant; component offsets in
          (z, x) cells: Ex (0, 1/2), Ey (0, 0), Ez (1/2, 0), Bx (1/2, 0),
          By (1/2, 1/2), Bz (0, 1/2); J like E.  float32 storage with one
          guard layer kept at zero (conducting walls).
  gather  linear (CIC) interpolation of every component at its own stagger,
          in float32 (the fields are float32): cell fractions are computed in
          float64 (half-staggered ones as f -/+ 1/2 from the cell fraction f,
          see _axis) and rounded to float32, then ((1-fz)((1-fx)a + fx b) +
          fz((1-fx)c + fx d)) in float32, result widened to float64.
  push    relativistic Boris rotation, then z += dt uz/gamma, x += dt ux/gamma.
  absorb  particles leaving [0, Nz) x [0, Nx) are removed (as in lbsim).
  deposit direct: J_c += q w v_c S(new position) at the component's stagger;
          float32 node weights, contribution ((v*scale)*wz)*wx with v rounded
          to float32 and a power-of-two scale; every node contribution is
          rounded to an integer (round half to even) and summed as
          integers -- order-independent, so the GPU's atomics reproduce it
          bit for bit; J = float32(sum / scale).
  field   B -= dt curl E ; E += dt (curl B - J) on interior nodes.
"""

from __future__ import annotations

import numpy as np

OFFSETS = {"Ex": (0.0, 0.5), "Ey": (0.0, 0.0), "Ez": (0.5, 0.0),
           "Bx": (0.5, 0.0), "By": (0.5, 0.5), "Bz": (0.0, 0.5)}
E_COMPS = ("Ex", "Ey", "Ez")
B_COMPS = ("Bx", "By", "Bz")


def new_fields(nz, nx):
    """float32 arrays (nz+2, nx+2), index [i+1, j+1] <-> cell (i, j)."""
    f = {k: np.zeros((nz + 2, nx + 2), dtype=np.float32) for k in OFFSETS}
    for k in ("Jx", "Jy", "Jz"):
        f[k] = np.zeros((nz + 2, nx + 2), dtype=np.float32)
    return f


def _axis(v, o):
    """One axis of the stencil (lbx_pic.cu axis_of): cell i = floor(v) and the
    exact fraction f = v - i; stagger 0 -> (i, f); stagger 1/2 -> the
    half-shifted stencil, (i, f - 1/2) when f >= 1/2 (exact) else
    (i - 1, f + 1/2).  Fractions are rounded to float32 last."""
    fl = np.floor(v)
    f = v - fl
    i = fl.astype(np.int64)
    if o == 0.0:
        return i, f.astype(np.float32)
    hi = f >= 0.5
    return np.where(hi, i, i - 1), np.where(hi, f - 0.5, f + 0.5).astype(np.float32)


def _stencil(z, x, oz, ox):
    i0, fz = _axis(z, oz)
    j0, fx = _axis(x, ox)
    return i0, j0, fz, fx


def gather(f, comp, z, x):
    oz, ox = OFFSETS[comp]
    i0, j0, fz, fx = _stencil(z, x, oz, ox)
    a = f[comp]
    g = lambda di, dj: a[i0 + 1 + di, j0 + 1 + dj]  # noqa: E731
    one = np.float32(1.0)
    gz, gx = one - fz, one - fx
    v = gz * (gx * g(0, 0) + fx * g(0, 1)) + fz * (gx * g(1, 0) + fx * g(1, 1))
    return v.astype(np.float64)


def current_scale(qw):
    """Power-of-two fixed-point scale: a single particle's largest node
    contribution (|qw|) maps to <= 2^20, so 1024-particle tile sums fit int32."""
    _, e = np.frexp(2.0 ** 20 / abs(qw))     # exact floor(log2(.)) = e - 1
    return float(2.0 ** (int(e) - 1))


def boris(uz, ux, uy, E, B, qm, dt):
    """E, B dicts of per-particle float64 values; returns new (uz, ux, uy)."""
    h = 0.5 * qm * dt
    mx, my, mz = ux + h * E["Ex"], uy + h * E["Ey"], uz + h * E["Ez"]
    g = np.sqrt(1.0 + mx * mx + my * my + mz * mz)
    ig = 1.0 / g
    tx, ty, tz = h * B["Bx"] * ig, h * B["By"] * ig, h * B["Bz"] * ig
    s = 2.0 / (1.0 + tx * tx + ty * ty + tz * tz)
    px, py, pz = mx + (my * tz - mz * ty), my + (mz * tx - mx * tz), mz + (mx * ty - my * tx)
    qx, qy, qz = mx + s * (py * tz - pz * ty), my + s * (pz * tx - px * tz), mz + s * (px * ty - py * tx)
    return qz + h * E["Ez"], qx + h * E["Ex"], qy + h * E["Ey"]


def deposit_acc(comp, z, x, val, scale, shape):
    """Integer fixed-point node sums of one current component (the exact
    quantity the GPU accumulates; summing these over ranks is exact)."""
    oz, ox = {"Jx": OFFSETS["Ex"], "Jy": OFFSETS["Ey"], "Jz": OFFSETS["Ez"]}[comp]
    i0, j0, fz, fx = _stencil(z, x, oz, ox)
    acc = np.zeros(shape, dtype=np.int64)
    one = np.float32(1.0)
    v32 = val.astype(np.float32)
    s32 = np.float32(scale)
    for di, wz in ((0, one - fz), (1, fz)):
        for dj, wx in ((0, one - fx), (1, fx)):
            q = np.rint(((v32 * s32) * wz) * wx).astype(np.int64)
            np.add.at(acc, (i0 + 1 + di, j0 + 1 + dj), q)
    return acc


def apply_current(f, comp, acc, scale):
    """J += float32(acc / scale) (lbx_pic.cu pic_current_kernel)."""
    f[comp] += (acc.astype(np.float64) / scale).astype(np.float32)


def deposit(f, comp, z, x, val, scale):
    apply_current(f, comp, deposit_acc(comp, z, x, val, scale, f[comp].shape), scale)


def push_particles(f, p, nz, nx, qm, dt):
    """Gather, Boris push, move, absorb: p (dict of float64 arrays z, x, uz,
    ux, uy) keeps the survivors in order; returns (keep mask, 1/gamma of the
    survivors)."""
    z, x = p["z"], p["x"]
    E = {k: gather(f, k, z, x) for k in E_COMPS}
    B = {k: gather(f, k, z, x) for k in B_COMPS}
    uz, ux, uy = boris(p["uz"], p["ux"], p["uy"], E, B, qm, dt)
    gam = np.sqrt(1.0 + ux * ux + uy * uy + uz * uz)
    ig = 1.0 / gam
    zn, xn = z + dt * uz * ig, x + dt * ux * ig
    keep = (zn >= 0) & (zn < nz) & (xn >= 0) & (xn < nx)
    for k, v in (("z", zn), ("x", xn), ("uz", uz), ("ux", ux), ("uy", uy)):
        p[k] = v[keep]
    return keep, ig[keep]


def current_accs(p, ig, qw, shape):
    """The three components' integer node sums of the particles p."""
    sc = current_scale(qw)
    return {comp: deposit_acc(comp, p["z"], p["x"], qw * u * ig, sc, shape)
            for comp, u in (("Jx", p["ux"]), ("Jy", p["uy"]), ("Jz", p["uz"]))}


def particle_step(f, p, nz, nx, qm, qw, dt):
    """Gather, Boris push, move, absorb, deposit.  p: dict of float64 arrays
    z, x, uz, ux, uy (modified: survivors only, order kept)."""
    keep, g = push_particles(f, p, nz, nx, qm, dt)
    sc = current_scale(qw)
    for comp, acc in current_accs(p, g, qw, f["Jx"].shape).items():
        apply_current(f, comp, acc, sc)
    return keep


def field_step(f, nz, nx, dt):
    """Yee update on interior nodes; guards stay zero; J consumed (zeroed)."""
    s = (slice(1, nz + 1), slice(1, nx + 1))
    Ex, Ey, Ez = (f[k].astype(np.float64) for k in E_COMPS)
    Bx, By, Bz = (f[k].astype(np.float64) for k in B_COMPS)
    # B -= dt curl E  (staggered differences; components at their offsets)
    nBx = Bx.copy()
    nBy = By.copy()
    nBz = Bz.copy()
    nBx[s] = Bx[s] + dt * (Ey[2:nz + 2, 1:nx + 1] - Ey[s])
    nBy[s] = By[s] - dt * ((Ex[2:nz + 2, 1:nx + 1] - Ex[s]) - (Ez[1:nz + 1, 2:nx + 2] - Ez[s]))
    nBz[s] = Bz[s] - dt * (Ey[1:nz + 1, 2:nx + 2] - Ey[s])
    nBx, nBy, nBz = (a.astype(np.float32).astype(np.float64) for a in (nBx, nBy, nBz))
    Jx, Jy, Jz = (f[k].astype(np.float64) for k in ("Jx", "Jy", "Jz"))
    nEx, nEy, nEz = Ex.copy(), Ey.copy(), Ez.copy()
    nEx[s] = Ex[s] + dt * (-(nBy[s] - nBy[0:nz, 1:nx + 1]) - Jx[s])
    nEy[s] = Ey[s] + dt * ((nBx[s] - nBx[0:nz, 1:nx + 1]) - (nBz[s] - nBz[1:nz + 1, 0:nx]) - Jy[s])
    nEz[s] = Ez[s] + dt * ((nBy[s] - nBy[1:nz + 1, 0:nx]) - Jz[s])
    for k, a in zip(B_COMPS, (nBx, nBy, nBz)):
        f[k][s] = a[s].astype(np.float32)
    for k, a in zip(E_COMPS, (nEx, nEy, nEz)):
        f[k][s] = a[s].astype(np.float32)
    for k in ("Jx", "Jy", "Jz"):
        f[k][:] = 0.0
