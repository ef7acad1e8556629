"""Kernel backend -- drop-in for lbsim.kernels (kernels.py:10-25).

Exposes the reference's module attributes ``advance_particles``,
``bin_particles`` and ``BACKEND``.  Both callables accept the reference's
host numpy arrays ([n, 2] float64) and return host numpy arrays, with the
work done by libLBX's sm_100a kernels (host->device copy, kernel,
device->host copy).  Given CUDA tensors they stay on the device.  There is
no CPU backend: without a CUDA device these raise RuntimeError.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as _dev

BACKEND = "cuda"

_ctxs: dict = {}


def _ctx(dev: torch.device) -> _dev.Context:
    key = dev.index or 0
    c = _ctxs.get(key)
    if c is None:
        c = _ctxs[key] = _dev.Context(f"cuda:{key}")
    return c


def _as_pairs(a, name):
    a = np.asarray(a)
    if a.dtype != np.float64:
        raise ValueError(f"Buffer dtype mismatch, expected 'double' for {name}")
    if a.ndim != 2 or a.shape[1] != 2:
        raise ValueError(f"{name} must have shape (n, 2), got {a.shape}")
    return np.ascontiguousarray(a)


def advance_particles(positions, velocities, extent_z, extent_x):
    """Move particles one step and drop those leaving [0, extent) on any
    axis; survivors keep their order (_kernels.pyx:12-35)."""
    if isinstance(positions, torch.Tensor):
        return _dev.advance_aos(_ctx(positions.device), positions.contiguous(),
                                velocities.contiguous(), extent_z, extent_x)
    pos = _as_pairs(positions, "positions")
    vel = _as_pairs(velocities, "velocities")
    if pos.shape != vel.shape:
        raise ValueError("positions and velocities differ in shape")
    _dev.require_cuda("cuda")
    dev = torch.device("cuda", torch.cuda.current_device())
    n = pos.shape[0]
    if n == 0:
        return np.empty((0, 2)), np.empty((0, 2))
    return advance_bin_host(pos, vel, extent_z, extent_x, dev=dev)[:2]


def advance_bin_host(pos, vel, extent_z, extent_x, box_size=None, nbz=0, nbx=0,
                     weights=(0.75, 0.25), out=None, dev=None):
    """Host arrays in, host arrays out, through lbx_advance_bin_host (chunked,
    both PCIe directions and the kernels overlapped).  With box_size also
    returns the survivors' per-box counts and heuristic cost.  `out` may
    supply (out_pos, out_vel) host buffers of shape (n, 2) (pinned = full
    speed)."""
    import ctypes as C

    from . import _lib

    dev = dev or torch.device("cuda", torch.cuda.current_device())
    n = pos.shape[0]
    op, ov = out if out is not None else (np.empty((n, 2)), np.empty((n, 2)))
    bin_ = box_size is not None
    counts = np.empty(int(nbz) * int(nbx), dtype=np.int64) if bin_ else None
    cost = np.empty(int(nbz) * int(nbx)) if bin_ else None
    m = C.c_int64()
    _lib.check(_lib.lib.lbx_advance_bin_host(
        _ctx(dev).handle, _lib.ptr(pos), _lib.ptr(vel), n, float(extent_z), float(extent_x),
        float(box_size or 1.0), int(nbz), int(nbx), float(weights[0]), float(weights[1]),
        _lib.ptr(op), _lib.ptr(ov), _lib.ptr(counts), _lib.ptr(cost), C.byref(m)))
    k = m.value
    return op[:k], ov[:k], counts, cost


def bin_particles(positions, box_size, nbz, nbx):
    """Per-box particle counts, box id = (int)(z/M)*nbx + (int)(x/M)
    (_kernels.pyx:38-47); int64, length nbz*nbx."""
    if isinstance(positions, torch.Tensor):
        return _dev.bin_aos(positions.contiguous(), box_size, nbz, nbx)
    pos = _as_pairs(positions, "positions")
    _dev.require_cuda("cuda")
    dev = torch.device("cuda", torch.cuda.current_device())
    if pos.shape[0] == 0:
        return np.zeros(int(nbz) * int(nbx), dtype=np.int64)
    return _dev.bin_aos(torch.from_numpy(pos).to(dev), box_size, nbz, nbx).cpu().numpy()
