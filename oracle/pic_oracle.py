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


# ----------------------------------------------------------------------------
# Charge-conserving (Esirkepov) deposition with shape order 1-3 (PAPER.md:235:
# the paper's runs use third-order particle shapes; deposition is ~50 % of
# the walltime).  Esirkepov, Comput. Phys. Commun. 135 (2001)
# 144, restated for the 2D (z, x) Yee grid with y invariant:
#   S0, S1   shape weights of the old / new position on a common window of
#            order+2 nodes per axis, DS = S1 - S0;
#   Wz = DSz (S0x + DSx/2),  Wx = DSx (S0z + DSz/2),
#   Wy = S0z S0x + (DSz S0x + S0z DSx)/2 + DSz DSx/3;
#   Jz(i+1/2, j) = -(q w / dt) sum_{i' <= i} Wz(i', j)   (Ez / Jz stagger),
#   Jx(i, j+1/2) = -(q w / dt) sum_{j' <= j} Wx(i, j')   (Ex / Jx stagger),
#   Jy(i, j)     = q w vy Wy.
# Then (rho1 - rho0)/dt + div J = 0 exactly (rho = q w S S on the nodes):
# Wz + Wx = S1z S1x - S0z S0x.  Fields are gathered with the same shape at
# each component's stagger.  fp64 throughout (the GPU kernel computes in
# float32 and is compared at a stated tolerance).
# ----------------------------------------------------------------------------

SHAPE_ORDERS = (1, 2, 3)


def shape_fn(order, d):
    """B-spline particle shape of the given order at node distance d."""
    a = np.abs(d)
    if order == 1:
        return np.where(a < 1.0, 1.0 - a, 0.0)
    if order == 2:
        return np.where(a <= 0.5, 0.75 - a * a,
                        np.where(a < 1.5, 0.5 * (1.5 - a) ** 2, 0.0))
    if order == 3:
        return np.where(a <= 1.0, 2.0 / 3.0 - a * a + 0.5 * a ** 3,
                        np.where(a < 2.0, (2.0 - a) ** 3 / 6.0, 0.0))
    raise ValueError(f"shape order must be 1, 2 or 3, got {order}")


def shape_base(pos, order):
    """Lowest node whose weight can be nonzero: floor(pos - (order+1)/2) + 1."""
    return np.floor(pos - 0.5 * (order + 1)).astype(np.int64) + 1


def window_weights(pos, base, order, width):
    """Weights S(base + k - pos), k = 0..width-1, shape (n, width)."""
    k = np.arange(width)
    return shape_fn(order, (base[:, None] + k[None, :]) - pos[:, None])


def gather_shaped(f, comp, z, x, order):
    """Shape-`order` gather of one component at its stagger (zero outside the
    stored nodes, i.e. beyond the one guard layer)."""
    oz, ox = OFFSETS[comp]
    zp, xp = z - oz, x - ox
    bz, bx = shape_base(zp, order), shape_base(xp, order)
    w = order + 1
    sz, sx = window_weights(zp, bz, order, w), window_weights(xp, bx, order, w)
    a = f[comp].astype(np.float64)
    nzg, nxg = a.shape
    out = np.zeros(z.shape[0])
    for di in range(w):
        ii = bz + di + 1
        okz = (ii >= 0) & (ii < nzg)
        for dj in range(w):
            jj = bx + dj + 1
            ok = okz & (jj >= 0) & (jj < nxg)
            v = np.zeros(z.shape[0])
            v[ok] = a[ii[ok], jj[ok]]
            out += sz[:, di] * sx[:, dj] * v
    return out


def esirkepov_current(z0, x0, z1, x1, vy, qw, dt, order, shape, pad):
    """fp64 Esirkepov current of particles moving (z0, x0) -> (z1, x1):
    dict Jz, Jx, Jy on padded node arrays of `shape` = (nz + 2 pad, nx + 2
    pad), index [i + pad, j + pad] <-> node (i, j) (Jz at i + 1/2, Jx at
    j + 1/2).  Contributions outside the padded arrays are dropped."""
    w = order + 2
    bz = shape_base(np.minimum(z0, z1), order)
    bx = shape_base(np.minimum(x0, x1), order)
    s0z, s1z = window_weights(z0, bz, order, w), window_weights(z1, bz, order, w)
    s0x, s1x = window_weights(x0, bx, order, w), window_weights(x1, bx, order, w)
    dsz, dsx = s1z - s0z, s1x - s0x
    wz = dsz[:, :, None] * (s0x + 0.5 * dsx)[:, None, :]
    wx = (s0z + 0.5 * dsz)[:, :, None] * dsx[:, None, :]
    wy = (s0z[:, :, None] * s0x[:, None, :] + 0.5 * dsz[:, :, None] * s0x[:, None, :]
          + 0.5 * s0z[:, :, None] * dsx[:, None, :] + dsz[:, :, None] * dsx[:, None, :] / 3.0)
    c = -(qw / dt)
    jz = c * np.cumsum(wz, axis=1)
    jx = c * np.cumsum(wx, axis=2)
    jy = (qw * vy)[:, None, None] * wy
    out = {k: np.zeros(shape) for k in ("Jz", "Jx", "Jy")}
    for di in range(w):
        ii = bz + di + pad
        for dj in range(w):
            jj = bx + dj + pad
            ok = (ii >= 0) & (ii < shape[0]) & (jj >= 0) & (jj < shape[1])
            for k, a in (("Jz", jz), ("Jx", jx), ("Jy", jy)):
                np.add.at(out[k], (ii[ok], jj[ok]), a[ok, di, dj])
    return out


def deposit_rho(z, x, qw, order, shape, pad):
    """Node charge density q w S(i - z) S(j - x) on the padded node arrays."""
    w = order + 1
    bz, bx = shape_base(z, order), shape_base(x, order)
    sz, sx = window_weights(z, bz, order, w), window_weights(x, bx, order, w)
    rho = np.zeros(shape)
    for di in range(w):
        ii = bz + di + pad
        for dj in range(w):
            jj = bx + dj + pad
            ok = (ii >= 0) & (ii < shape[0]) & (jj >= 0) & (jj < shape[1])
            np.add.at(rho, (ii[ok], jj[ok]), qw * sz[ok, di] * sx[ok, dj])
    return rho


def push_particles_shaped(f, p, nz, nx, qm, dt, order):
    """Gather (shape `order`), Boris, move, absorb; returns (keep mask, old
    z, old x of the survivors, 1/gamma of the survivors)."""
    z, x = p["z"], p["x"]
    E = {k: gather_shaped(f, k, z, x, order) for k in E_COMPS}
    B = {k: gather_shaped(f, k, z, x, order) for k in B_COMPS}
    uz, ux, uy = boris(p["uz"], p["ux"], p["uy"], E, B, qm, dt)
    ig = 1.0 / np.sqrt(1.0 + ux * ux + uy * uy + uz * uz)
    zn, xn = z + dt * uz * ig, x + dt * ux * ig
    keep = (zn >= 0) & (zn < nz) & (xn >= 0) & (xn < nx)
    z0, x0 = z[keep], x[keep]
    for k, v in (("z", zn), ("x", xn), ("uz", uz), ("ux", ux), ("uy", uy)):
        p[k] = v[keep]
    return keep, z0, x0, ig[keep]


def particle_step_esirkepov(f, p, nz, nx, qm, qw, dt, order):
    """Shape-`order` gather, Boris, move, absorb, Esirkepov deposit of the
    survivors into f's J arrays (one guard layer: contributions further out
    are dropped).  Returns the keep mask."""
    keep, z0, x0, ig = push_particles_shaped(f, p, nz, nx, qm, dt, order)
    j = esirkepov_current(z0, x0, p["z"], p["x"], p["uy"] * ig, qw, dt, order,
                          f["Jx"].shape, 1)
    for k in ("Jx", "Jy", "Jz"):
        f[k] += j[k].astype(np.float32)
    return keep


def field_energy(f):
    """0.5 sum(E^2 + B^2) over the stored nodes (cell volume 1)."""
    return 0.5 * sum(float(np.sum(f[k].astype(np.float64) ** 2)) for k in OFFSETS)


def kinetic_energy(p, mass_w):
    """sum w m (gamma - 1) (c = 1) for macro weight x mass `mass_w`."""
    g = np.sqrt(1.0 + p["uz"] ** 2 + p["ux"] ** 2 + p["uy"] ** 2)
    return float(mass_w * np.sum(g - 1.0))
