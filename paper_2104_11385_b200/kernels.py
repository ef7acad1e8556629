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
    dev = _dev.require_cuda("cuda")
    dev = torch.device("cuda", torch.cuda.current_device())
    if pos.shape[0] == 0:
        return np.empty((0, 2)), np.empty((0, 2))
    p, v = _dev.advance_aos(_ctx(dev), torch.from_numpy(pos).to(dev),
                            torch.from_numpy(vel).to(dev), extent_z, extent_x)
    return p.cpu().numpy(), v.cpu().numpy()


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
