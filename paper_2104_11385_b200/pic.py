"""2D3V electromagnetic PIC step on the device.

The paper's per-box work is a WarpX PIC step: field gather, Lorentz (Boris)
push, current deposition, field solve.  The
reference only models it as ballistic motion, so this physics is the
builder's own (checked against oracle/pic_oracle.py, parity unpinned).  The
per-box counts / GpuClock tallies it produces feed the same balancer.
See include/lbx.h (lbx_pic_step) for conventions.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import Context, _stream, require_cuda

FIELD_NAMES = ("Ex", "Ey", "Ez", "Bx", "By", "Bz")
CURRENT_NAMES = ("Jx", "Jy", "Jz")


@dataclass
class PicState:
    z: torch.Tensor
    x: torch.Tensor
    uz: torch.Tensor
    ux: torch.Tensor
    uy: torch.Tensor
    n: int
    fields: dict
    nz: int
    nx: int

    spare: tuple = None     # sorted mode: output buffers (z, x, uz, ux, uy), swapped each step

    @classmethod
    def create(cls, pos, u, nz, nx, device="cuda:0"):
        dev = require_cuda(device)
        pos = np.asarray(pos, dtype=np.float64).reshape(-1, 2)
        u = np.asarray(u, dtype=np.float64).reshape(-1, 3)   # (uz, ux, uy)
        n = pos.shape[0]
        arrs = []
        for col in (pos[:, 0], pos[:, 1], u[:, 0], u[:, 1], u[:, 2]):
            t = torch.zeros(n + 2, dtype=torch.float64, device=dev)
            t[:n].copy_(torch.from_numpy(np.ascontiguousarray(col)))
            arrs.append(t)
        fields = {k: torch.zeros((nz + 2, nx + 2), dtype=torch.float32, device=dev)
                  for k in FIELD_NAMES + CURRENT_NAMES}
        return cls(*arrs, n=n, fields=fields, nz=nz, nx=nx)

    def particles(self):
        n = self.n
        return {k: getattr(self, k)[:n].cpu().numpy() for k in ("z", "x", "uz", "ux", "uy")}

    def field_arrays(self):
        return {k: v.cpu().numpy() for k, v in self.fields.items()}


def pic_sync(ctx: Context, st: PicState) -> int:
    """After steps / sorts run with sync=False: wait for the device and read
    the particle count back into st.n."""
    st.n = ctx.count()
    return st.n


def _device_count(ctx: Context, st: PicState, sync: bool):
    """The context's device count must be this state's before a kernel runs:
    set from st.n unless (sync=False) this state's own previous step / sort
    left it there (then st.n is only an upper bound).  Call pic_sync before
    running another state on the same context."""
    live = getattr(ctx, "_pic_live", None)
    if sync or live is None or live() is not st:
        ctx.set_count(st.n)
    ctx._pic_live = weakref.ref(st)


def pic_sort(ctx: Context, st: PicState, tiled: bool = False, sync: bool = True):
    """Counting sort of the particles by cell (lbx_pic_sort) into the spare
    buffers, which the state then swaps in.  Every few in-place steps this
    restores the cell order the deposit's register runs feed on.  tiled=True
    sorts by a tile-major key and records the tile ranges that
    pic_step(tiled=True) works on.  sync=False: as pic_step(sync=False)."""
    dev = ctx.device
    names = ("z", "x", "uz", "ux", "uy")
    _device_count(ctx, st, sync)
    cap = st.z.numel()
    if st.spare is None or st.spare[0].numel() != cap:
        st.spare = tuple(torch.zeros(cap, dtype=torch.float64, device=dev) for _ in names)
    a = _lib.PicArgs()
    a.z, a.x, a.uz, a.ux, a.uy = (_lib.ptr(getattr(st, k)) for k in names)
    a.nz, a.nx = st.nz, st.nx
    a.flags = _lib.LBX_PIC_TILED if tiled else 0
    for i, t in enumerate(st.spare):
        a.out[i] = _lib.ptr(t)
    _lib.check(_lib.lib.lbx_pic_sort(ctx.handle, C.byref(a), _stream(dev)))
    old = tuple(getattr(st, k) for k in names)
    for k, t in zip(names, st.spare):
        setattr(st, k, t)
    st.spare = old
    ctx._pic_sorted = None


def pic_step(ctx: Context, st: PicState, box_size: int, q_over_m: float, q_times_w: float,
             dt: float, weights=(0.75, 0.25), clock=False, field_solve=True, sort=False,
             gather=None, stable=False, tiled=False, fast=False, shape_order=0, sync=True):
    """One PIC step; returns per-box counts / cost / clock and n.

    sort=False: in place; absorbed particles' slots are filled from the tail
    (O(absorbed)), or with stable=True the order is kept (stable compaction).
    sort=True: sort-on-write -- results land in a second buffer set grouped by
    each particle's cell at the start of the step, which the state then
    swaps in (order within a cell is not deterministic; values are).
    tiled=True: in place, one CTA per 16x16-cell tile with the field patch
    and the current in shared memory, on the tile ranges of the last
    pic_sort(tiled=True) -- the sparse-plasma path.
    fast=True (in place, also tiled): tolerance mode (LBX_PIC_FAST) -- float32
    Boris increment with FMA and MUFU rsqrt/rcp, FMA gathers; agrees with
    the fp64 oracle within the tolerances tests/test_gpu_pic_fast.py states,
    not bit for bit.
    shape_order=1..3 (in place): charge-conserving Esirkepov deposition
    with B-spline shapes of that order and the same-order gather (the
    paper's order 3); tolerance mode, checked against
    oracle/pic_oracle.py esirkepov_current (tests/test_gpu_pic_esirkepov.py).
    sync=False: no host round trip -- the device keeps the particle count
    from this state's previous step / sort on this context (set from st.n
    on the first call; st.n stays an upper bound), nothing is read back and
    None is returned; pic_sync() ends such a sequence.  Back-to-back steps
    then time the device alone."""
    dev = ctx.device
    nbz, nbx = st.nz // box_size, st.nx // box_size
    nb = nbz * nbx
    counts = torch.empty(nb, dtype=torch.int64, device=dev)
    cost = torch.empty(nb, dtype=torch.float64, device=dev)
    clk = torch.zeros(nb, dtype=torch.int64, device=dev)
    nout = torch.zeros(2, dtype=torch.int64, device=dev)
    _device_count(ctx, st, sync)
    a = _lib.PicArgs()
    a.z, a.x, a.uz, a.ux, a.uy = (_lib.ptr(getattr(st, k)) for k in ("z", "x", "uz", "ux", "uy"))
    for i, k in enumerate(FIELD_NAMES):
        a.fields[i] = _lib.ptr(st.fields[k])
    for i, k in enumerate(CURRENT_NAMES):
        a.current[i] = _lib.ptr(st.fields[k])
    a.nz, a.nx, a.box_size = st.nz, st.nx, int(box_size)
    a.q_over_m, a.q_times_w, a.dt = float(q_over_m), float(q_times_w), float(dt)
    a.w_particle, a.w_cell = float(weights[0]), float(weights[1])
    a.flags = (_lib.LBX_STEP_CLOCK if clock else 0) | (0 if field_solve else
                                                        _lib.LBX_PIC_NO_FIELD_SOLVE)
    if stable and not sort:
        a.flags |= _lib.LBX_PIC_STABLE_ORDER
    if gather is not None:     # "quad" | "direct" (default: by particles per cell)
        a.flags |= {"quad": _lib.LBX_PIC_QUAD, "direct": _lib.LBX_PIC_DIRECT}[gather]
    if tiled:
        if sort:
            raise ValueError("tiled steps run in place (sort=False)")
        a.flags |= _lib.LBX_PIC_TILED
    if fast:
        if sort:
            raise ValueError("fast (tolerance) steps run in place")
        a.flags |= _lib.LBX_PIC_FAST
    if shape_order:
        if sort or tiled:
            raise ValueError("shape_order > 0 steps run in place, untiled")
        a.shape_order = int(shape_order)
    a.counts_out, a.cost_out, a.clk_out = _lib.ptr(counts), _lib.ptr(cost), _lib.ptr(clk)
    a.n_out, a.err_out = _lib.ptr(nout), _lib.ptr(nout[1:])
    names = ("z", "x", "uz", "ux", "uy")
    if sort:
        # The library keeps the cell slots of its last sorted output and
        # recognises that output by address; a new state can reuse a freed
        # buffer's address, so resynchronise unless this state (unmodified
        # since: torch's version counter) produced the last sorted output.
        last = getattr(ctx, "_pic_sorted", None)
        if last is None or last[0]() is not st or last[1] != st.z._version:
            a.flags |= _lib.LBX_PIC_RESYNC
        cap = st.z.numel()
        if st.spare is None or st.spare[0].numel() != cap:
            st.spare = tuple(torch.zeros(cap, dtype=torch.float64, device=dev) for _ in names)
        for i, t in enumerate(st.spare):
            a.out[i] = _lib.ptr(t)
    _lib.check(_lib.lib.lbx_pic_step(ctx.handle, C.byref(a), _stream(dev)))
    if sort:
        old = tuple(getattr(st, k) for k in names)
        for k, t in zip(names, st.spare):
            setattr(st, k, t)
        st.spare = old
        ctx._pic_sorted = (weakref.ref(st), st.z._version)
    else:
        ctx._pic_sorted = None
    if not sync:
        return None
    h = nout.cpu().numpy()
    if h[1]:
        raise ValueError(f"{int(h[1])} particles fell outside the box grid")
    st.n = int(h[0])
    return dict(counts=counts.cpu().numpy(), cost=cost.cpu().numpy(),
                clock=clk.cpu().numpy().view(np.uint64), n=st.n)
