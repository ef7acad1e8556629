"""Device-resident particle state and the stream-ordered libLBX device calls.

torch is used only as the allocator and stream provider: every kernel is
libLBX's own sm_100a code reached through the C ABI (include/lbx.h).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr

_PAD = 2  # spare slots so 16-byte pair loads never run off the allocation


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def require_cuda(device="cuda:0") -> torch.device:
    dev = torch.device(device)
    if dev.type != "cuda" or not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2104_11385_b200 runs on a CUDA device only (sm_100a); "
            "there is no CPU fallback")
    return dev


class Context:
    """Owns an lbx_ctx: look-back workspace + device-resident step state."""

    def __init__(self, device="cuda:0", capacity: int = 0):
        self.device = require_cuda(device)
        h = C.c_void_p()
        check(lib.lbx_ctx_create(C.byref(h), self.device.index or 0, int(capacity)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib.lbx_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_count(self, n: int):
        check(lib.lbx_ctx_set_count(self.handle, int(n), _stream(self.device)))

    def count(self) -> int:
        out = C.c_int64()
        check(lib.lbx_ctx_get_count(self.handle, C.byref(out), _stream(self.device)))
        return out.value

    def set_grid(self, ctas: int):
        check(lib.lbx_ctx_set_grid(self.handle, int(ctas)))


@dataclass
class ParticleState:
    """SoA float64 particle state in HBM: z, x, vz, vx (capacity >= n + 2).

    Slices [0:n] are live; the fused step compacts survivors in place.
    """

    z: torch.Tensor
    x: torch.Tensor
    vz: torch.Tensor
    vx: torch.Tensor
    n: int

    @classmethod
    def empty(cls, capacity: int, device="cuda:0") -> "ParticleState":
        dev = require_cuda(device)
        cap = int(capacity) + _PAD
        mk = lambda: torch.zeros(cap, dtype=torch.float64, device=dev)  # noqa: E731
        return cls(mk(), mk(), mk(), mk(), 0)

    @classmethod
    def from_numpy(cls, pos, vel, device="cuda:0", capacity=None) -> "ParticleState":
        pos = np.asarray(pos, dtype=np.float64).reshape(-1, 2)
        vel = np.asarray(vel, dtype=np.float64).reshape(-1, 2)
        n = pos.shape[0]
        st = cls.empty(n if capacity is None else capacity, device)
        st.load(pos, vel)
        return st

    def load(self, pos, vel):
        n = pos.shape[0]
        for dst, src in ((self.z, pos[:, 0]), (self.x, pos[:, 1]),
                         (self.vz, vel[:, 0]), (self.vx, vel[:, 1])):
            dst[:n].copy_(torch.from_numpy(np.ascontiguousarray(src)))
        self.n = n

    def to_numpy(self):
        n = self.n
        pos = np.stack([self.z[:n].cpu().numpy(), self.x[:n].cpu().numpy()], axis=1)
        vel = np.stack([self.vz[:n].cpu().numpy(), self.vx[:n].cpu().numpy()], axis=1)
        return pos, vel


def push_step(ctx: Context, st: ParticleState, extent_z, extent_x, box_size, nbz, nbx,
              weights=(0.75, 0.25), clock=False, sync=True):
    """One fused step on `st` (in place).  Returns counts/cost/clock/n when
    sync=True (host copies), else the device output tensors."""
    dev = ctx.device
    nb = nbz * nbx
    counts = torch.empty(nb, dtype=torch.int64, device=dev)
    cost = torch.empty(nb, dtype=torch.float64, device=dev)
    clk = torch.zeros(nb, dtype=torch.int64, device=dev)
    n_out = torch.empty(2, dtype=torch.int64, device=dev)
    ctx.set_count(st.n)
    args = _lib.StepArgs(
        ptr(st.z), ptr(st.x), ptr(st.vz), ptr(st.vx), float(extent_z), float(extent_x),
        float(box_size), int(nbz), int(nbx), float(weights[0]), float(weights[1]),
        float(box_size) * float(box_size), _lib.LBX_STEP_CLOCK if clock else 0,
        ptr(counts), ptr(cost), ptr(clk), ptr(n_out), ptr(n_out[1:]))
    check(lib.lbx_push_step(ctx.handle, C.byref(args), _stream(dev)))
    if not sync:
        return dict(counts=counts, cost=cost, clock=clk, n=n_out)
    n_host = n_out.cpu().numpy()
    if n_host[1] != 0:
        raise ValueError(f"{int(n_host[1])} survivors fall outside the box grid")
    st.n = int(n_host[0])
    return dict(counts=counts.cpu().numpy(), cost=cost.cpu().numpy(),
                clock=clk.cpu().numpy().view(np.uint64), n=st.n)


def advance_aos(ctx: Context, pos: torch.Tensor, vel: torch.Tensor, extent_z, extent_x):
    """Reference-layout advance on device tensors [n,2] -> (pos', vel')."""
    n = pos.shape[0]
    out_p = torch.empty((n + 1, 2), dtype=torch.float64, device=pos.device)
    out_v = torch.empty((n + 1, 2), dtype=torch.float64, device=pos.device)
    m = torch.empty(1, dtype=torch.int64, device=pos.device)
    check(lib.lbx_advance_particles(ctx.handle, ptr(pos), ptr(vel), n, float(extent_z),
                                    float(extent_x), ptr(out_p), ptr(out_v), ptr(m),
                                    _stream(pos.device)))
    k = int(m.item())
    return out_p[:k], out_v[:k]


def bin_aos(pos: torch.Tensor, box_size, nbz, nbx) -> torch.Tensor:
    """Reference-layout per-box counts on a device tensor [n,2]."""
    nb = int(nbz) * int(nbx)
    counts = torch.empty(max(nb, 1), dtype=torch.int64, device=pos.device)
    err = torch.zeros(1, dtype=torch.int64, device=pos.device)
    check(lib.lbx_bin_particles(ptr(pos), pos.shape[0], float(box_size), int(nbz), int(nbx),
                                ptr(counts), ptr(err), _stream(pos.device)))
    if int(err.item()):
        raise ValueError(f"{int(err.item())} positions fall outside the "
                         f"{nbz}x{nbx} box grid")
    return counts[:nb]
