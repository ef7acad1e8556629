"""Multi-GPU runtime: box ownership -> GPU.

One process per GPU.  Rank r holds the particles of the boxes it owns
(``owner[b] == r``).  Per step, on every rank:

  1. libLBX exchange step: push + absorb + per-box counts / GpuClock tally of
     everything this rank pushed; a survivor whose box is owned elsewhere is
     staged as a 6-double record for its owner and compacted out locally.
  2. all-reduce(sum) of the per-box counts (and clock tally): every box's
     particles were pushed by exactly one rank, so the sum is the exact
     global vector -- bit-identical to a single-process run.
  3. box-crossing exchange: all-to-all of per-destination counts, then of the
     records (NCCL over NVLink on B200; gloo in the CPU tests), unpack.
  4. every rank runs the same host step (lbx_lb_step: cost vector,
     efficiency, knapsack/SFC attempt, adoption gate, walltime columns) on
     the same vector, so all ranks agree with no broadcast (PAPER.md:146,155
     gathers to a root and broadcasts; replicated deterministic remapping
     replaces that).
  5. on adoption: every rank stages the particles of the boxes it lost
     (lbx_partition) and the same all-to-all migrates them -- the
     redistribution the reference only models (workload.py:332-337).

Parity: metrics, cost trace and mappings equal the reference run with
ranks = world size; the particle multiset equals it (local order differs).
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _lib
from .errors import ConfigError
from .workload import (RunResult, StepMetrics, box_array_for, initial_mapping,
                       kick_velocities, policy_kind, sample_blob, sim_config)

REC = _lib.RECORD_DOUBLES


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------

class TorchComm:
    """torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_reduce_sum(self, t: torch.Tensor):
        self.dist.all_reduce(t, group=self.group)

    def all_reduce_max(self, t: torch.Tensor):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)

    def exchange_counts(self, send_counts: torch.Tensor) -> torch.Tensor:
        recv = torch.empty_like(send_counts)
        self.dist.all_to_all_single(recv, send_counts, group=self.group)
        return recv

    def exchange_records(self, send: torch.Tensor, sc: list, rc: list) -> torch.Tensor:
        recv = torch.empty((sum(rc), REC), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(recv, send, rc, sc, group=self.group)
        return recv

    def exchange_values(self, send: torch.Tensor, sc: list, rc: list) -> torch.Tensor:
        """All-to-all of a flat tensor with per-peer element counts."""
        recv = torch.empty(sum(rc), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(recv, send, rc, sc, group=self.group)
        return recv

    def barrier(self):
        self.dist.barrier(group=self.group)

    def device_ids(self, dev: int) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, int(dev), group=self.group)
        return out

    def share_peer(self, ptr: int, handle: bytes) -> tuple:
        """Every rank's peer buffer mapped into this process: (pointers,
        pointers this process opened and must close)."""
        hs = [None] * self.world
        self.dist.all_gather_object(hs, bytes(handle), group=self.group)
        ptrs, opened = [], []
        for r, h in enumerate(hs):
            if r == self.rank:
                ptrs.append(int(ptr))
                continue
            q = C.c_void_p()
            buf = (C.c_ubyte * 64).from_buffer_copy(h)
            if _lib.lib.lbx_peer_open(buf, C.byref(q)) != 0:
                ptrs.append(None)          # the caller agrees on failure collectively
                continue
            ptrs.append(int(q.value))
            opened.append(int(q.value))
        return ptrs, opened


class ThreadComm:
    """In-process communicator for `world` ranks run as threads (tests on a
    single GPU).  Create one shared state with ThreadComm.shared(world)."""

    @staticmethod
    def shared(world: int) -> dict:
        return {"world": world, "bar": threading.Barrier(world), "slot": [None] * world}

    def __init__(self, shared: dict, rank: int):
        self.s = shared
        self.rank = rank
        self.world = shared["world"]

    def _swap(self, value):
        self.s["slot"][self.rank] = value
        self.s["bar"].wait()
        vals = list(self.s["slot"])
        self.s["bar"].wait()
        return vals

    def all_reduce_sum(self, t: torch.Tensor):
        vals = self._swap(t.detach().cpu().clone())
        total = vals[0].clone()
        for v in vals[1:]:
            total += v
        t.copy_(total.to(t.device))

    def all_reduce_max(self, t: torch.Tensor):
        vals = self._swap(t.detach().cpu().clone())
        total = vals[0].clone()
        for v in vals[1:]:
            total = torch.maximum(total, v)
        t.copy_(total.to(t.device))

    def exchange_counts(self, send_counts: torch.Tensor) -> torch.Tensor:
        vals = self._swap(send_counts.detach().cpu().clone())
        return torch.stack([v[self.rank] for v in vals]).to(send_counts.device)

    def exchange_records(self, send: torch.Tensor, sc: list, rc: list) -> torch.Tensor:
        chunks = list(torch.split(send.detach().cpu(), sc))
        vals = self._swap(chunks)
        out = torch.cat([v[self.rank] for v in vals]) if vals else send[:0].cpu()
        return out.reshape(-1, REC).to(send.device)

    def exchange_values(self, send: torch.Tensor, sc: list, rc: list) -> torch.Tensor:
        chunks = list(torch.split(send.detach().cpu(), sc))
        vals = self._swap(chunks)
        out = torch.cat([v[self.rank] for v in vals])
        assert out.numel() == sum(rc)
        return out.to(send.device)

    def barrier(self):
        # A device barrier, as NCCL's is: this rank's queued work (e.g. the
        # unpack of its receive buffer and the cursor reset) completes before
        # any peer passes, so a peer's next push cannot race it.
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.current_stream().synchronize()
        self.s["bar"].wait()

    def device_ids(self, dev: int) -> list:
        return self._swap(int(dev))

    def share_peer(self, ptr: int, handle: bytes) -> tuple:
        return self._swap(int(ptr)), []     # one address space: raw pointers


# ---------------------------------------------------------------------------
# device engine (libLBX)
# ---------------------------------------------------------------------------

class DeviceEngine:
    """This rank's particles in HBM and the libLBX exchange kernels."""

    def __init__(self, cfg, rank, world, device, pos, kick, capacity, clock):
        from . import device as D

        self.dev = D.require_cuda(device)
        self.D = D
        self.rank, self.world = rank, world
        self.nbz, self.nbx = box_array_for(cfg).grid_shape
        self.nb = self.nbz * self.nbx
        self.ez, self.ex = float(cfg.domain_extent[0]), float(cfg.domain_extent[1])
        self.m = float(cfg.box_size)
        self.clock = clock
        cap = int(capacity) + 2
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.z, self.x = torch.zeros(cap, **f64), torch.zeros(cap, **f64)
        self.vz, self.vx = torch.zeros(cap, **f64), torch.zeros(cap, **f64)
        self.kvz = self.kvx = None
        n = int(pos.shape[0])
        p = torch.as_tensor(pos).to(self.dev)
        self.z[:n].copy_(p[:, 0])
        self.x[:n].copy_(p[:, 1])
        if kick is not None:
            k = torch.as_tensor(kick).to(self.dev)
            self.kvz, self.kvx = torch.zeros(cap, **f64), torch.zeros(cap, **f64)
            self.kvz[:n].copy_(k[:, 0])
            self.kvx[:n].copy_(k[:, 1])
        self.n = n
        self.capacity = int(capacity)
        self.stage = torch.empty((cap, REC), **f64)
        self.stage_dest = torch.empty(cap, dtype=torch.int32, device=self.dev)
        self.removed = torch.empty(cap, dtype=torch.int64, device=self.dev)
        self.send_counts = torch.zeros(world, dtype=torch.int64, device=self.dev)
        self.owner = torch.zeros(self.nb, dtype=torch.int32, device=self.dev)
        self.counts = torch.zeros(self.nb, dtype=torch.int64, device=self.dev)
        self.cost = torch.zeros(self.nb, **f64)
        self.clk = torch.zeros(self.nb, dtype=torch.int64, device=self.dev)
        self.nout = torch.zeros(2, dtype=torch.int64, device=self.dev)
        self.ctx = D.Context(self.dev, capacity=cap)
        self.launches = 0   # libLBX kernel launches issued (for gpu_launches)
        self.p2p = False
        self.parity = 0

    # -- fused exchange over peer memory ---------------------------------
    def enable_p2p(self, comm):
        """Peer-memory exchange: every rank exposes two receive buffers
        (step parity) + two cursors; the push / partition kernels write
        emigrant records straight into the destination's buffer (remote
        atomics + stores over NVLink / NVSwitch), replacing staging, the
        counts all-to-all, the grouping kernel and the record all-to-all.
        Single-rank convenience: DistributedSimulation runs the phases with
        agreement between them (p2p_alloc / p2p_connect)."""
        self.p2p_alloc()
        ptrs, opened = comm.share_peer(self._peer_own, self._peer_handle)
        if any(q is None for q in ptrs):
            self._peer_opened = list(opened)
            self.p2p_release()
            raise RuntimeError("cudaIpcOpenMemHandle failed for a peer buffer")
        self.p2p_connect(ptrs, opened)

    def p2p_alloc(self):
        """Local phase 1: this rank's receive buffers (may fail)."""
        nrec = self.capacity + 2
        self._peer_per = nrec * REC * 8
        ptr, handle = C.c_void_p(), (C.c_ubyte * 64)()
        _lib.check(_lib.lib.lbx_peer_alloc(2 * self._peer_per + 64, C.byref(ptr), handle))
        self._peer_own = int(ptr.value)
        self._peer_handle = bytes(handle)
        self._peer_opened = []

    def p2p_connect(self, ptrs, opened):
        """Local phase 2 (after the collective handle exchange): device tables
        of every rank's buffers and cursors."""
        per, nrec = self._peer_per, self.capacity + 2
        self._peer_opened = list(opened)
        i64 = dict(dtype=torch.int64, device=self.dev)
        self.peer_recv = [torch.tensor([b + par * per for b in ptrs], **i64) for par in (0, 1)]
        self.peer_cursor = [torch.tensor([b + 2 * per + 8 * par for b in ptrs], **i64)
                            for par in (0, 1)]
        self.peer_cap = nrec
        self.recv_base = [self._peer_own + par * per for par in (0, 1)]
        self.cursor = [torch.as_tensor(_DevArray(self._peer_own + 2 * per + 8 * par, 1, "<i8"),
                                       device=self.dev) for par in (0, 1)]
        self.stage = torch.empty((1, REC), dtype=torch.float64, device=self.dev)
        self.stage_dest = torch.empty(1, dtype=torch.int32, device=self.dev)
        self.p2p = True

    def p2p_release(self):
        """Undo p2p_alloc / an opened mapping (failure path, no kernels ran)."""
        for q in getattr(self, "_peer_opened", []):
            _lib.lib.lbx_peer_close(C.c_void_p(q))
        self._peer_opened = []
        if getattr(self, "_peer_own", None):
            _lib.lib.lbx_peer_free(C.c_void_p(self._peer_own))
            self._peer_own = None

    def close_p2p(self):
        if not self.p2p:
            return
        torch.cuda.synchronize(self.dev)
        for q in self._peer_opened:
            _lib.lib.lbx_peer_close(C.c_void_p(q))
        self._peer_opened = []
        self.cursor = None
        _lib.lib.lbx_peer_free(C.c_void_p(self._peer_own))
        self.p2p = False

    def unpack_peer(self, parity: int, m: int):
        """Append the m records other ranks wrote into this rank's receive
        buffer `parity`, then reset its cursor (stream-ordered)."""
        if self.n + m > self.capacity:
            raise MemoryError(f"rank {self.rank}: {self.n + m} particles exceed capacity "
                              f"{self.capacity}")
        if m:
            _lib.check(_lib.lib.lbx_unpack(C.c_void_p(self.recv_base[parity]), m, self.n,
                                           _lib.ptr(self.z), _lib.ptr(self.x), _lib.ptr(self.vz),
                                           _lib.ptr(self.vx), _lib.ptr(self.kvz),
                                           _lib.ptr(self.kvx), self.D._stream(self.dev)))
            self.launches += 1
        self.cursor[parity].zero_()
        self.n += m

    # -- pipelined loop (device-resident counts, no host round trip) ----
    def begin_async(self):
        self.ctx.set_count(self.n)     # the device count takes over from here
        _lib.check(_lib.lib.lbx_ctx_set_upper(self.ctx.handle, self.capacity + 2))

    def end_async(self):
        self.n = self.ctx.count()      # the device count is authoritative again

    def push_async(self, wp, wc):
        """The exchange push on the device live count (no set_count), then
        the hole filling of the removed slots, all stream-ordered."""
        self.send_counts.zero_()
        args = _lib.StepArgs(
            _lib.ptr(self.z), _lib.ptr(self.x), _lib.ptr(self.vz), _lib.ptr(self.vx),
            self.ez, self.ex, self.m, self.nbz, self.nbx, float(wp), float(wc),
            self.m * self.m, _lib.LBX_STEP_CLOCK if self.clock else 0,
            _lib.ptr(self.counts), _lib.ptr(self.cost), _lib.ptr(self.clk),
            _lib.ptr(self.nout), _lib.ptr(self.nout[1:]))
        ex = self._ex()
        st = self.D._stream(self.dev)
        _lib.check(_lib.lib.lbx_push_step_exchange(self.ctx.handle, C.byref(args), C.byref(ex), st))
        _lib.check(_lib.lib.lbx_fill_holes_dev(
            self.ctx.handle, _lib.ptr(self.z), _lib.ptr(self.x), _lib.ptr(self.vz),
            _lib.ptr(self.vx), _lib.ptr(self.kvz), _lib.ptr(self.kvx), _lib.ptr(self.removed),
            self.capacity + 2, self.ez, self.ex, st))
        self.launches += 5   # stream kernel, fill mark / move / done
        return self.counts, self.clk, self.send_counts, self.nout

    def unpack_peer_async(self, parity: int):
        _lib.check(_lib.lib.lbx_unpack_peer_dev(
            self.ctx.handle, C.c_void_p(self.recv_base[parity]),
            C.c_void_p(int(self.cursor[parity].data_ptr())), self.capacity,
            _lib.ptr(self.z), _lib.ptr(self.x), _lib.ptr(self.vz), _lib.ptr(self.vx),
            _lib.ptr(self.kvz), _lib.ptr(self.kvx), self.D._stream(self.dev)))
        self.launches += 2

    def _ex(self):
        a = _lib.ExchangeArgs(
            _lib.ptr(self.owner), self.rank, self.world, _lib.ptr(self.stage),
            _lib.ptr(self.stage_dest), self.capacity + 2, _lib.ptr(self.send_counts),
            _lib.ptr(self.kvz), _lib.ptr(self.kvx), _lib.ptr(self.removed), self.capacity + 2)
        if self.p2p:
            a.peer_recv = _lib.ptr(self.peer_recv[self.parity])
            a.peer_cursor = _lib.ptr(self.peer_cursor[self.parity])
            a.peer_recv_cap = self.peer_cap
        return a

    def set_owner(self, owner: np.ndarray):
        self.owner.copy_(torch.from_numpy(np.asarray(owner, dtype=np.int32)))

    def kick(self):
        if self.kvz is not None:
            self.vz, self.vx, self.kvz, self.kvx = self.kvz, self.kvx, None, None

    def push(self, wp, wc):
        self.send_counts.zero_()
        self.ctx.set_count(self.n)
        args = _lib.StepArgs(
            _lib.ptr(self.z), _lib.ptr(self.x), _lib.ptr(self.vz), _lib.ptr(self.vx),
            self.ez, self.ex, self.m, self.nbz, self.nbx, float(wp), float(wc),
            self.m * self.m, _lib.LBX_STEP_CLOCK if self.clock else 0,
            _lib.ptr(self.counts), _lib.ptr(self.cost), _lib.ptr(self.clk),
            _lib.ptr(self.nout), _lib.ptr(self.nout[1:]))
        ex = self._ex()
        _lib.check(_lib.lib.lbx_push_step_exchange(self.ctx.handle, C.byref(args), C.byref(ex),
                                                   self.D._stream(self.dev)))
        self.launches += 3   # set_count, stream kernel, compaction
        return self.counts, self.clk, self.send_counts, self.nout

    def partition(self):
        self.send_counts.zero_()
        self.ctx.set_count(self.n)
        ex = self._ex()
        _lib.check(_lib.lib.lbx_partition(
            self.ctx.handle, _lib.ptr(self.z), _lib.ptr(self.x), _lib.ptr(self.vz),
            _lib.ptr(self.vx), self.ez, self.ex, self.m, self.nbz, self.nbx, C.byref(ex),
            _lib.ptr(self.nout), self.D._stream(self.dev)))
        self.launches += 3
        return self.send_counts, self.nout

    def commit(self, nout_host):
        """Adopt the local count left by push/partition (host copy of nout)
        and compact: O(removed) hole filling (local order is not kept)."""
        if int(nout_host[1]) != 0:
            raise ValueError("particles outside the box grid or staging overflow "
                             f"(code {int(nout_host[1])})")
        n_new = int(nout_host[0])
        _lib.check(_lib.lib.lbx_fill_holes(
            self.ctx.handle, _lib.ptr(self.z), _lib.ptr(self.x), _lib.ptr(self.vz),
            _lib.ptr(self.vx), _lib.ptr(self.kvz), _lib.ptr(self.kvx), _lib.ptr(self.removed),
            self.n - n_new, n_new, self.D._stream(self.dev)))
        self.launches += 3
        self.n = n_new

    def pack(self, sc: list) -> torch.Tensor:
        total = int(sum(sc))
        send = torch.empty((total, REC), dtype=torch.float64, device=self.dev)
        if total:
            cur = torch.tensor(np.concatenate(([0], np.cumsum(sc)[:-1])), dtype=torch.int64,
                               device=self.dev)
            _lib.check(_lib.lib.lbx_group_by_dest(_lib.ptr(self.stage), _lib.ptr(self.stage_dest),
                                                  total, self.world, _lib.ptr(cur), _lib.ptr(send),
                                                  self.D._stream(self.dev)))
            self.launches += 1
        return send

    def unpack(self, recv: torch.Tensor):
        m = int(recv.shape[0])
        if self.n + m > self.capacity:
            raise MemoryError(f"rank {self.rank}: {self.n + m} particles exceed capacity "
                              f"{self.capacity}")
        if m:
            recv = recv.contiguous()
            _lib.check(_lib.lib.lbx_unpack(_lib.ptr(recv), m, self.n, _lib.ptr(self.z),
                                           _lib.ptr(self.x), _lib.ptr(self.vz), _lib.ptr(self.vx),
                                           _lib.ptr(self.kvz), _lib.ptr(self.kvx),
                                           self.D._stream(self.dev)))
            self.launches += 1
        self.n += m

    def state(self):
        n = self.n
        pos = torch.stack([self.z[:n], self.x[:n]], 1).cpu().numpy()
        vel = torch.stack([self.vz[:n], self.vx[:n]], 1).cpu().numpy()
        return pos, vel


class _DevArray:
    """A device pointer owned by libLBX, viewed as a torch tensor
    (__cuda_array_interface__, no copy)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


# ---------------------------------------------------------------------------
# guard-cell (halo) planning for the box-decomposed PIC
# ---------------------------------------------------------------------------

def cell_owner_map(owner, grid_shape, box_size: int) -> np.ndarray:
    """Owner rank of every cell (nz, nx) from the per-box owner vector."""
    nbz, nbx = grid_shape
    o = np.asarray(owner, dtype=np.int64).reshape(nbz, nbx)
    return np.repeat(np.repeat(o, box_size, axis=0), box_size, axis=1)


def dilate(mask: np.ndarray, k: int) -> np.ndarray:
    """Chebyshev dilation of a boolean cell mask by k cells (clipped to the grid)."""
    out = mask
    for _ in range(k):
        g = out.copy()
        g[1:, :] |= out[:-1, :]
        g[:-1, :] |= out[1:, :]
        h = g.copy()
        h[:, 1:] |= g[:, :-1]
        h[:, :-1] |= g[:, 1:]
        out = h
    return out


def halo_plan(src_cells: np.ndarray, dst_cells: np.ndarray, rank: int, world: int,
              src_grow: int, dst_grow: int):
    """Cells this rank exchanges with every peer: send[q] = S(rank) & D(q),
    recv[q] = S(q) & D(rank), with S(x) = own_src(x) grown by src_grow cells
    and D(x) = own_dst(x) grown by dst_grow (flat row-major cell indices,
    ascending, so both ends of a pair list the same cells in the same
    order).  send[rank] = recv[rank] = empty."""
    S = [dilate(src_cells == r, src_grow) for r in range(world)]
    D = [dilate(dst_cells == r, dst_grow) for r in range(world)]
    send, recv = [], []
    for q in range(world):
        if q == rank:
            send.append(np.zeros(0, dtype=np.int64))
            recv.append(np.zeros(0, dtype=np.int64))
            continue
        send.append(np.flatnonzero(S[rank] & D[q]).astype(np.int64))
        recv.append(np.flatnonzero(S[q] & D[rank]).astype(np.int64))
    return send, recv


def bbox(mask: np.ndarray):
    """(r0, r1, c0, c1) of the True cells, or an empty box."""
    rows, cols = np.flatnonzero(mask.any(axis=1)), np.flatnonzero(mask.any(axis=0))
    if rows.size == 0:
        return (2 ** 31 - 1, -2 ** 31, 2 ** 31 - 1, -2 ** 31)
    return (int(rows[0]), int(rows[-1]), int(cols[0]), int(cols[-1]))


class PicHalo:
    """One rank's exchange plan for an owner map (device index tensors):
    current: the cell-centric int64 rows Jc[cell][16] of cells within one
    cell of both ranks' boxes (a particle deposits at its new cell, at most
    one cell outside its box; a node needs the rows of the cells around
    it) -- summed into the receiver's rows;  fields: the owner's E, B
    values of its cells within two cells of the receiver's boxes (the Yee
    update of the owned cells reads one cell around them, the gather one) --
    copied over the receiver's stale values.  Bytes per step scale with the
    off-rank faces, not with the grid."""

    def __init__(self, owner, grid_shape, box_size, nz, nx, rank, world, dev, order=0):
        self.owner = np.asarray(owner, dtype=np.int64).copy()
        self.order = int(order)
        cells = cell_owner_map(owner, grid_shape, box_size)
        # field guard ring: the gather reaches one cell (CIC) or `order` - 1
        # cells (B-spline order K) beyond the particle's cell, the Yee update
        # of the owned cells one
        self.guard = max(2, self.order)
        if self.order:
            # Esirkepov: node-centric sums on the padded node grid of
            # lbx_pic_esk_current_view (guard G nodes around the cells; a
            # padding node belongs to its nearest cell's owner).  A rank's
            # particles deposit within 4 nodes of their boxes (window base
            # one node below the cell after a downward move, K + 2 nodes up).
            G = ESK_GUARD
            padded = np.pad(cells, G, mode="edge")
            js, jr = halo_plan(padded, padded, rank, world, self.order + 1, 1)
        else:
            js, jr = halo_plan(cells, cells, rank, world, 1, 1)
        fs, fr = halo_plan(cells, cells, rank, world, 0, self.guard)
        self.j_send_n = [int(a.size) for a in js]
        self.j_recv_n = [int(a.size) for a in jr]
        self.f_send_n = [int(a.size) for a in fs]
        self.f_recv_n = [int(a.size) for a in fr]
        t = lambda a: torch.from_numpy(np.concatenate(a)).to(dev)  # noqa: E731
        self.j_send, self.j_recv = t(js), t(jr)
        pad = lambda c: (c // nx + 1) * (nx + 2) + (c % nx + 1)  # noqa: E731 (cell -> padded node)
        self.f_send = t([pad(a) for a in fs])
        self.f_recv = t([pad(a) for a in fr])
        self.box = torch.tensor(bbox(dilate(cells == rank, 1)), dtype=torch.int32, device=dev)
        self.bytes_j = (3 if self.order else 16) * 8 * sum(self.j_send_n)
        self.bytes_f = 6 * 4 * sum(self.f_send_n)


ESK_GUARD = 4   # lbx_pic_esk_current_view's guard nodes (kEskG in lbx_pic.cu)


def field_sync_plan(old_owner, new_owner, grid_shape, box_size, nx, rank, world, dev,
                    guard=2):
    """Adoption: every rank's new guard region (own_new grown by `guard`) from
    the cells' previous owners (who hold their current values)."""
    old = cell_owner_map(old_owner, grid_shape, box_size)
    new = cell_owner_map(new_owner, grid_shape, box_size)
    fs, fr = halo_plan(old, new, rank, world, 0, guard)
    pad = lambda c: (c // nx + 1) * (nx + 2) + (c % nx + 1)  # noqa: E731
    t = lambda a: torch.from_numpy(np.concatenate(a)).to(dev)  # noqa: E731
    return (t([pad(a) for a in fs]), [int(a.size) for a in fs], t([pad(a) for a in fr]),
            [int(a.size) for a in fr])


class PicEngine(DeviceEngine):
    """This rank's share of a box-decomposed PIC run (pic.py physics).

    Particles: the rank's boxes (z, x, uz, ux, uy in HBM).  Fields: each rank
    keeps grid-sized arrays but only its own cells (and a two-cell guard
    ring) are current: after the particle step (current deferred, exact
    integers, LBX_PIC_DEFER_CURRENT) the ranks exchange the current rows of
    the cells along their shared faces (PicHalo: one all-to-all, sizes known
    from the owner map on every rank), finish (node gather over the rank's
    region, Yee update), then exchange the owners' E, B values of the
    two-cell guard rings.  Bytes per step scale with the off-rank faces
    (the reference's face model, workload.py:324-327, decomposition.py:71-81).
    Integer sums are order independent, so every rank's own cells are
    bit-identical to one GPU.  On adoption the new owners first receive the
    fields of their new guard regions from the previous owners.  Emigrants
    and adoption-time migration reuse the 6-double records: (z, x, uz, ux,
    kick_z, kick_x) before the kick (uy is 0 then), (z, x, uz, ux, uy, 0)
    after it."""

    def __init__(self, cfg, rank, world, device, pos, kick, capacity, clock, pic=None):
        from .pic import CURRENT_NAMES, FIELD_NAMES
        from .workload import PIC_DEFAULTS
        super().__init__(cfg, rank, world, device, pos, kick, capacity, clock)
        self.pic = dict(PIC_DEFAULTS, **(pic or {}))
        self.order = int(self.pic.get("shape_order", 0))   # 0: CIC; 1-3: Esirkepov
        # cell-sort the rank's particles every `resort` steps after the kick
        # (lbx_pic_sort: the deposit's runs / held blocks follow cell order;
        # emigrant unpacking and hole filling scramble it) -- 0: never
        self.resort = int(self.pic.get("resort", 0))
        # tolerance mode (LBX_PIC_FAST, the pipelined kernel on dense plasmas)
        self.fast = bool(self.pic.get("fast", False))
        self._sortbuf = None
        self._steps = 0
        nz, nx = cfg.domain_extent
        self.nz, self.nx = int(nz), int(nx)
        cap = self.capacity + 2
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.uy = torch.zeros(cap, **f64)
        self.spare = torch.zeros(cap, **f64)
        self.kicked = self.kvz is None
        if self.kicked:
            self.kvz, self.kvx = self.uy, self.spare
        self.fields = {k: torch.zeros((nz + 2, nx + 2), dtype=torch.float32, device=self.dev)
                       for k in FIELD_NAMES + CURRENT_NAMES}
        self.field_names, self.current_names = FIELD_NAMES, CURRENT_NAMES
        self.comm = None
        self.time_step = False      # bench_lb: CUDA events around the particle kernels
        self.last_ms = 0.0
        self.nout2 = torch.zeros(2, dtype=torch.int64, device=self.dev)
        self.halo = None
        self.halo_bytes = 0          # bytes sent by this rank's last step's exchanges

    def attach_comm(self, comm):
        self.comm = comm

    def set_owner(self, owner: np.ndarray):
        owner = np.asarray(owner, dtype=np.int64)
        if self.halo is not None and not np.array_equal(owner, self.halo.owner):
            self.field_sync(self.halo.owner, owner)
        super().set_owner(owner)
        if self.halo is None or not np.array_equal(owner, self.halo.owner):
            self.halo = PicHalo(owner, (self.nbz, self.nbx), int(self.m), self.nz, self.nx,
                                self.rank, self.world, self.dev, order=self.order)

    def _field_exchange(self, send_idx, sc, recv_idx, rc):
        names = self.field_names
        send = torch.stack([self.fields[k].view(-1).index_select(0, send_idx) for k in names],
                           1)
        recv = self.comm.exchange_values(send.reshape(-1), [6 * k for k in sc],
                                         [6 * k for k in rc]).view(-1, 6)
        for c, k in enumerate(names):
            self.fields[k].view(-1).index_copy_(0, recv_idx, recv[:, c].contiguous())
        return 6 * 4 * sum(sc)

    def field_sync(self, old_owner, new_owner):
        """Adoption: the new guard regions' fields from the previous owners."""
        plan = field_sync_plan(old_owner, new_owner, (self.nbz, self.nbx), int(self.m),
                               self.nx, self.rank, self.world, self.dev,
                               guard=max(2, self.order))
        self._field_exchange(*plan)

    def kick(self):
        if not self.kicked:     # momenta u = v_kick / dt, as Simulation(physics="pic")
            dt = self.pic["dt"]
            self.vz, self.vx = self.kvz.div_(dt), self.kvx.div_(dt)
            self.kvz, self.kvx = self.uy, self.spare
            self.kicked = True

    def _args(self, flags):
        a = _lib.PicArgs()
        a.z, a.x, a.uz, a.ux, a.uy = (_lib.ptr(t) for t in (self.z, self.x, self.vz, self.vx,
                                                             self.uy))
        for i, k in enumerate(self.field_names):
            a.fields[i] = _lib.ptr(self.fields[k])
        for i, k in enumerate(self.current_names):
            a.current[i] = _lib.ptr(self.fields[k])
        a.nz, a.nx, a.box_size = self.nz, self.nx, int(self.m)
        a.q_over_m, a.q_times_w = float(self.pic["q_over_m"]), float(self.pic["q_times_w"])
        a.dt = float(self.pic["dt"])
        a.flags = flags
        a.shape_order = self.order
        return a

    def push(self, wp, wc):
        self.local_step(wp, wc)
        self.current_sum_finish()
        send_counts, nout = self.partition()
        return self.counts, self.clk, send_counts, nout

    def _resort(self, stream):
        """Counting sort of the rank's particles by cell into the spare
        buffers, then swap (after the kick: (z, x, uz, ux, uy) is the whole
        particle record; kvz aliases uy from then on)."""
        names = ("z", "x", "vz", "vx", "uy")
        cap = self.z.numel()
        if self._sortbuf is None or self._sortbuf[0].numel() != cap:
            self._sortbuf = [torch.zeros(cap, dtype=torch.float64, device=self.dev)
                             for _ in names]
        a = self._args(0)
        for i, t in enumerate(self._sortbuf):
            a.out[i] = _lib.ptr(t)
        _lib.check(_lib.lib.lbx_pic_sort(self.ctx.handle, C.byref(a), stream))
        old = [getattr(self, k) for k in names]
        for k, t in zip(names, self._sortbuf):
            setattr(self, k, t)
        self._sortbuf = old
        self.kvz = self.uy
        self.launches += 4   # count, scan reduce, scan apply, scatter

    def local_step(self, wp, wc):
        """The rank's particle kernels: PIC step with the current deferred."""
        stream = self.D._stream(self.dev)
        self.ctx.set_count(self.n)
        if self.resort and self.kicked and self._steps % self.resort == 0 and self.n:
            self._resort(stream)
        self._steps += 1
        a = self._args((_lib.LBX_STEP_CLOCK if self.clock else 0) | _lib.LBX_PIC_DEFER_CURRENT
                       | (_lib.LBX_PIC_FAST if self.fast and not self.order else 0))
        a.w_particle, a.w_cell = float(wp), float(wc)
        a.counts_out, a.cost_out, a.clk_out = (_lib.ptr(self.counts), _lib.ptr(self.cost),
                                               _lib.ptr(self.clk))
        a.n_out, a.err_out = _lib.ptr(self.nout2), _lib.ptr(self.nout2[1:])
        if self.time_step:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
        _lib.check(_lib.lib.lbx_pic_step(self.ctx.handle, C.byref(a), stream))
        if self.time_step:
            ev[1].record()
        self.launches += 6   # set_count, quad, push, compaction, (scan), current view
        h = self.nout2.cpu().numpy()
        if self.time_step:
            self.last_ms = ev[0].elapsed_time(ev[1])
        if h[1]:
            raise ValueError(f"{int(h[1])} particles fell outside the box grid")
        self.n = int(h[0])

    def current_sum_finish(self):
        """Guard-cell exchange of the current, node gather + Yee update over
        the rank's region, then the guard rings' fields from their owners."""
        self.current_sum()
        self.finish()
        h = self.halo
        self.halo_bytes += self._field_exchange(h.f_send, h.f_send_n, h.f_recv, h.f_recv_n)

    def finish(self):
        _lib.check(_lib.lib.lbx_pic_finish(self.ctx.handle, C.byref(self._args(0)),
                                           self.D._stream(self.dev)))
        self.launches += 4   # current, zero, B, E

    def current_sum(self):
        """Integer current rows of the shared-face cells, summed into each
        receiver's rows; the node gather then covers the rank's cells grown
        by one (every nonzero row lies there).  Esirkepov (shape_order > 0):
        the node sums near the shared faces, summed into the receivers'."""
        if self.order:
            return self._esk_current_sum()
        jc_p, cells, box_p = C.c_void_p(), C.c_int64(), C.c_void_p()
        _lib.check(_lib.lib.lbx_pic_current_view(self.ctx.handle, C.byref(jc_p), C.byref(cells),
                                                 C.byref(box_p)))
        h = self.halo
        jc = torch.as_tensor(_DevArray(jc_p.value, cells.value * 16, "<i8"),
                             device=self.dev).view(-1, 16)
        send = jc.index_select(0, h.j_send)
        recv = self.comm.exchange_values(send.reshape(-1), [16 * k for k in h.j_send_n],
                                         [16 * k for k in h.j_recv_n])
        jc.index_add_(0, h.j_recv, recv.view(-1, 16))
        box = torch.as_tensor(_DevArray(box_p.value, 4, "<i4"), device=self.dev)
        box.copy_(h.box)
        self.halo_bytes = 16 * 8 * sum(h.j_send_n)

    def _esk_current_sum(self):
        j_p, stride, guard = C.c_void_p(), C.c_int64(), C.c_int32()
        _lib.check(_lib.lib.lbx_pic_esk_current_view(self.ctx.handle, C.byref(j_p),
                                                     C.byref(stride), C.byref(guard)))
        if guard.value != ESK_GUARD:
            raise RuntimeError(f"libLBX Esirkepov guard {guard.value} != {ESK_GUARD}")
        h = self.halo
        j = torch.as_tensor(_DevArray(j_p.value, 3 * stride.value, "<i8"),
                            device=self.dev).view(3, -1)
        send = j.index_select(1, h.j_send).t().contiguous()          # [k, 3]
        recv = self.comm.exchange_values(send.reshape(-1), [3 * k for k in h.j_send_n],
                                         [3 * k for k in h.j_recv_n])
        j.index_add_(1, h.j_recv, recv.view(-1, 3).t())
        self.halo_bytes = 3 * 8 * sum(h.j_send_n)

    def unpack(self, recv: torch.Tensor):
        n0 = self.n
        super().unpack(recv)
        if not self.kicked:     # uy is not carried before the kick: it is 0
            self.uy[n0:self.n].zero_()

    def unpack_peer(self, parity: int, m: int):
        n0 = self.n
        super().unpack_peer(parity, m)
        if not self.kicked:
            self.uy[n0:self.n].zero_()

    def state(self):
        n = self.n
        return {k: t[:n].cpu().numpy() for k, t in (("z", self.z), ("x", self.x), ("uz", self.vz),
                                                    ("ux", self.vx), ("uy", self.uy))}

    def field_arrays(self):
        return {k: v.cpu().numpy() for k, v in self.fields.items()}


# ---------------------------------------------------------------------------
# driver
# ---------------------------------------------------------------------------

def box_ids_host(pos: np.ndarray, box_size: int, nbx: int) -> np.ndarray:
    """(int)(z/M)*nbx + (int)(x/M) on the host (setup only: selecting each
    rank's initial particles), IEEE division then truncation."""
    return (np.trunc(pos[:, 0] / float(box_size)).astype(np.int64) * nbx
            + np.trunc(pos[:, 1] / float(box_size)).astype(np.int64))


class DistributedSimulation:
    """One rank of a box-decomposed run (see module docstring)."""

    def __init__(self, cfg, policy, provider, *, comm=None, engine_factory=None,
                 positions=None, kick=None, device=None, capacity=None,
                 record_counts=False, replicas=1, physics="surrogate", pic=None,
                 exchange="auto", pipeline=True):
        self.comm = comm or TorchComm()
        self.rank, self.world = self.comm.rank, self.comm.world
        if cfg.n_ranks != self.world:
            raise ConfigError(f"scenario has {cfg.n_ranks} ranks but the job has {self.world}")
        if provider.device_kind < 0 or provider.device_kind > 3:
            raise ConfigError(f"provider {provider.kind!r} is not supported by the native loop")
        self.cfg, self.policy, self.provider = cfg, policy, provider
        self.ba = box_array_for(cfg)
        nbz, nbx = self.ba.grid_shape
        # `replicas`: the particle set is tiled that many times (identical
        # copies evolve identically; used to fill a B200 with the C2 set).
        pos = sample_blob(cfg) if positions is None else np.asarray(positions)
        self.n_init = int(pos.shape[0]) * replicas
        ids = box_ids_host(pos, cfg.box_size, nbx)
        counts0 = replicas * np.bincount(ids, minlength=nbz * nbx).astype(np.int64)
        self.initial_owner = np.array(initial_mapping(cfg, self.ba, counts0).owner)
        mine = self.initial_owner[ids] == self.rank
        if cfg.kick.step < cfg.total_steps and kick is None:
            kick = kick_velocities(pos, cfg)
        kick_local = None if kick is None or cfg.kick.step >= cfg.total_steps else kick[mine]
        local = pos[mine]
        if replicas > 1:
            local = np.tile(local, (replicas, 1))
            kick_local = None if kick_local is None else np.tile(kick_local, (replicas, 1))
        cap = capacity if capacity is not None else self.n_init
        if physics not in ("surrogate", "pic"):
            raise ConfigError(f"unknown physics {physics!r}")
        factory = engine_factory or (PicEngine if physics == "pic" else DeviceEngine)
        if physics == "pic":
            self.engine = factory(cfg, self.rank, self.world, device, local, kick_local, cap,
                                  provider.device_kind == 3, pic=pic)
            self.engine.attach_comm(self.comm)
        else:
            self.engine = factory(cfg, self.rank, self.world, device, local, kick_local, cap,
                                  provider.device_kind == 3)
        self.engine.set_owner(self.initial_owner)
        self.exchange = self._choose_exchange(exchange)
        if self.exchange == "p2p":
            self._enable_p2p(exchange == "p2p")
        # pipelined loop: the GPU runs the next step while the host does this
        # step's LB bookkeeping; needs the fused exchange (device-resident
        # counts) and no capacity model (an OOM halt must stop at its step)
        self.pipeline = bool(pipeline and self.exchange == "p2p"
                             and hasattr(self.engine, "push_async")
                             and physics == "surrogate" and cfg.capacity_particles is None)
        self.conf = sim_config(cfg, policy, provider)
        h = C.c_void_p()
        own = np.ascontiguousarray(self.initial_owner, dtype=np.int64)
        _lib.check(_lib.lib.lbx_lb_create(C.byref(h), C.byref(self.conf), _lib.ptr(own)))
        self.lb = h
        T, nb = cfg.total_steps, self.ba.n_boxes
        o = {k: np.zeros(T) for k in ("eff_before", "eff_after", "compute_max", "comm_max",
                                      "gather", "redistribute", "walltime")}
        for k in ("adopted", "attempted", "oom"):
            o[k] = np.zeros(T, dtype=np.uint8)
        o["max_rank_particles"] = np.zeros(T, dtype=np.int64)
        o["n_alive"] = np.zeros(T, dtype=np.int64)
        o["cost_trace"] = np.zeros((T, nb))
        o["count_trace"] = np.zeros((T, nb), dtype=np.int64) if record_counts else None
        o["adopt_steps"] = np.zeros(T, dtype=np.int64)
        o["adopt_owners"] = np.zeros((T, nb), dtype=np.int64)
        o["owner"] = own.copy()
        self.out = o
        self.souts = _lib.SimOutputs(
            *(_lib.ptr(o.get(k)) for k in ("eff_before", "eff_after", "adopted", "attempted",
                                           "compute_max", "comm_max", "gather", "redistribute",
                                           "walltime", "max_rank_particles", "oom", "n_alive",
                                           "cost_trace", "count_trace", "clock_trace", "owner",
                                           "adopt_steps", "adopt_owners")),
            None, 0, 0, 0)
        self.done = 0
        self.halted = False
        self.moved = np.zeros(T, dtype=np.int64)   # particles migrated on adoption
        # measured redistribution cost (policy.measured_migration)
        self.measure_mig = bool(getattr(policy, "measured_migration", False))
        self.mig_log = []            # per adoption: step, moved, migration ms, push ms, ratio
        self.mig_ratio = float(getattr(policy, "migration_ratio", 0.0))
        self._push_ev = None

    def _choose_exchange(self, exchange):
        """p2p (fused exchange over peer memory) when the engine supports it
        and every rank's GPU can access every other's; else collectives."""
        if exchange not in ("auto", "p2p", "nccl"):
            raise ConfigError(f"exchange must be auto, p2p or nccl; got {exchange!r}")
        capable = (hasattr(self.engine, "enable_p2p") and hasattr(self.comm, "share_peer")
                   and getattr(self.engine, "dev", None) is not None
                   and self.engine.dev.type == "cuda")
        ok = False
        if capable and exchange != "nccl":
            devs = self.comm.device_ids(self.engine.dev.index)
            yes = C.c_int32()
            ok = True
            for d in devs:
                _lib.check(_lib.lib.lbx_peer_can_access(int(self.engine.dev.index), int(d),
                                                        C.byref(yes)))
                ok = ok and bool(yes.value)
            flags = torch.tensor([1 if ok else 0], dtype=torch.int64, device=self.engine.dev)
            self.comm.all_reduce_sum(flags)     # every rank must agree
            ok = int(flags.item()) == self.world
        if exchange == "p2p" and not ok:
            raise ConfigError("exchange='p2p' needs CUDA engines with peer access between all ranks")
        return "p2p" if ok else "nccl"

    def _enable_p2p(self, required):
        """Map the peers' receive buffers in two phases with a collective
        agreement after each (allocation; handle exchange + mapping): if any
        rank fails (IPC not permitted in the container, no peer mapping, out
        of memory) every rank falls back to the collective exchange."""
        def agree(ok):
            flag = torch.tensor([1 if ok else 0], dtype=torch.int64, device=self.engine.dev)
            self.comm.all_reduce_sum(flag)
            return int(flag.item()) == self.world

        err = None
        try:
            self.engine.p2p_alloc()
            ok = True
        except Exception as e:   # noqa: BLE001 -- agreed on below
            ok, err = False, e
        if agree(ok):
            ptrs, opened = self.comm.share_peer(self.engine._peer_own, self.engine._peer_handle)
            ok = all(q is not None for q in ptrs)
            self.engine._peer_opened = list(opened)
            if not ok:
                err = RuntimeError("cudaIpcOpenMemHandle failed for a peer buffer")
            if agree(ok):
                self.engine.p2p_connect(ptrs, opened)
                return
        self.comm.barrier()
        self.engine.p2p_release()
        if required:
            raise ConfigError(f"exchange='p2p' could not map peer memory: {err}")
        self.exchange = "nccl"
        self.p2p_error = str(err) if err else "a peer rank failed"

    def close(self, collective=True):
        """Release native state.  With the peer-memory exchange every rank's
        buffers are mapped by the others, so by default close is collective
        (all ranks call it together); collective=False when the caller knows
        no rank runs any more (e.g. thread-ranks closed one after another)."""
        if getattr(self, "engine", None) is not None and getattr(self.engine, "p2p", False):
            if collective:
                self.comm.barrier()        # peers may still map this rank's buffers
            self.engine.close_p2p()
            if collective:
                self.comm.barrier()
        if getattr(self, "lb", None):
            _lib.lib.lbx_lb_destroy(self.lb)
            self.lb = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _push_events(self):
        """CUDA events bracketing this step's push (measured migration)."""
        if not self.measure_mig or not torch.cuda.is_available():
            return None
        return [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]

    def _timed_migration(self, step, fn):
        """Run a migration; with policy.measured_migration, time it (device
        synchronised wall time, max over ranks) against the last push and
        return the new per-particle price (pushes per moved particle) for
        the adoption gate, else None."""
        import time
        if not self.measure_mig:
            return fn(), None
        dev = self.engine.dev
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        moved = fn()
        torch.cuda.synchronize(dev)
        mig_ms = 1e3 * (time.perf_counter() - t0)
        ev = self._push_ev
        push_ms = ev[0].elapsed_time(ev[1]) if ev is not None else 0.0
        v = torch.tensor([mig_ms, push_ms, float(self.engine.n), float(moved)],
                         dtype=torch.float64, device=dev)
        tot = v.clone()
        self.comm.all_reduce_max(v)
        self.comm.all_reduce_sum(tot)
        mig_ms, push_ms, n_max = float(v[0]), float(v[1]), float(v[2])
        moved_all = int(tot[3])
        ratio = None
        if moved_all > 0 and push_ms > 0 and n_max > 0:
            r = (mig_ms / moved_all) / (push_ms / n_max)
            ratio = r if not self.mig_log else 0.5 * (self.mig_ratio + r)
        self.mig_log.append({"step": int(step), "moved": moved_all, "migration_ms": mig_ms,
                             "push_ms": push_ms, "ratio": ratio})
        return moved, ratio

    def _set_mig_ratio(self, ratio):
        if ratio is not None:
            self.mig_ratio = float(ratio)
            _lib.check(_lib.lib.lbx_lb_set_migration_ratio(self.lb, self.mig_ratio))

    def _records(self, sc, rc):
        """All-to-all of the staged records given host split sizes."""
        send = self.engine.pack(sc)
        recv = self.comm.exchange_records(send, sc, rc)
        self.engine.unpack(recv)

    def _migrate_p2p(self, step):
        """Adoption-time migration over peer memory: the partition kernel
        writes the lost boxes' particles into their new owners' buffers
        (parity (step+1)&1 -- the buffer the NEXT step's push writes its
        emigrants into); the all-reduce orders every sender before the reads;
        the barrier (a device barrier on every communicator: NCCL's, and
        ThreadComm's syncs the rank's stream first) keeps the next step's
        pushes out until every rank has drained that buffer and reset its
        cursor."""
        par = (step + 1) & 1
        self.engine.parity = par
        send_counts, nout = self.engine.partition()
        total = send_counts.sum().reshape(1)
        self.comm.all_reduce_sum(total)
        h = torch.cat([nout, total, self.engine.cursor[par]]).cpu().numpy()
        self.engine.commit(h[:2])
        self.engine.unpack_peer(par, int(h[3]))
        self.comm.barrier()
        return int(send_counts.sum().item())

    def _migrate(self):
        """Adoption-time redistribution: stage the particles of lost boxes,
        one counts exchange + one host copy, then the record all-to-all."""
        send_counts, nout = self.engine.partition()
        total = send_counts.sum().reshape(1)
        self.comm.all_reduce_sum(total)
        recv_counts = self.comm.exchange_counts(send_counts)
        h = torch.cat([nout, total, send_counts, recv_counts]).cpu().numpy()
        self.engine.commit(h[:2])
        w = self.world
        sc, rc = [int(v) for v in h[3:3 + w]], [int(v) for v in h[3 + w:3 + 2 * w]]
        if int(h[2]):
            self._records(sc, rc)
        return sum(sc)

    def run(self, first=None, last=None):
        """Steps [first, last).  Per step: push (no host sync), one all-reduce
        of [counts, clock tally, global emigrant count], one all-to-all of
        per-destination counts, ONE device->host copy, then the record
        all-to-all only if some rank has emigrants, then the host LB step.
        With the fused peer-memory exchange the loop is pipelined instead
        (`_run_pipelined`)."""
        cfg = self.cfg
        first = self.done if first is None else first
        last = cfg.total_steps if last is None else last
        w = getattr(self.provider, "weights", None)
        wp, wc = (w.w_particle, w.w_cell) if w else (0.75, 0.25)
        clock = self.provider.device_kind == 3
        if self.pipeline:
            return self._run_pipelined(first, last, wp, wc, clock)
        nb, W = self.ba.n_boxes, self.world
        adopted, halt = C.c_int32(), C.c_int32()
        for step in range(first, last):
            if self.halted:
                break
            if step == cfg.kick.step:
                self.engine.kick()
            p2p = self.exchange == "p2p"
            if p2p:
                self.engine.parity = step & 1
            ev = self._push_events()
            if ev:
                ev[0].record()
            counts, clk, send_counts, nout = self.engine.push(wp, wc)
            if ev:
                ev[1].record()
                self._push_ev = ev
            parts = [counts, clk] if clock else [counts]
            red = torch.cat(parts + [send_counts.sum().reshape(1)])
            self.comm.all_reduce_sum(red)   # p2p: also orders every sender's kernel first
            k = len(parts) * nb
            if p2p:
                h = torch.cat([red, nout, self.engine.cursor[step & 1]]).cpu().numpy()
            else:
                recv_counts = self.comm.exchange_counts(send_counts)
                h = torch.cat([red, nout, send_counts, recv_counts]).cpu().numpy()
            ch = np.ascontiguousarray(h[:nb], dtype=np.int64)
            kh = np.ascontiguousarray(h[nb:2 * nb]).view(np.uint64) if clock else None
            emigrants = int(h[k])
            self.engine.commit(h[k + 1:k + 3])
            if p2p:
                self.engine.unpack_peer(step & 1, int(h[k + 3]))
            else:
                sc = [int(v) for v in h[k + 3:k + 3 + W]]
                rc = [int(v) for v in h[k + 3 + W:k + 3 + 2 * W]]
                if emigrants:
                    self._records(sc, rc)
            _lib.check(_lib.lib.lbx_lb_step(self.lb, step, _lib.ptr(ch), _lib.ptr(kh),
                                            int(ch.sum()), C.byref(self.souts),
                                            C.byref(adopted), C.byref(halt)))
            if adopted.value:
                owner = np.empty(nb, dtype=np.int64)
                _lib.check(_lib.lib.lbx_lb_owner(self.lb, _lib.ptr(owner)))
                self.engine.set_owner(owner)
                self.moved[step], ratio = self._timed_migration(
                    step, (lambda: self._migrate_p2p(step)) if p2p else self._migrate)
                self._set_mig_ratio(ratio)      # prices the next adoptions (same on every rank)
            self.done = step + 1
            if halt.value:
                self.halted = True
        return self

    def _run_pipelined(self, first, last, wp, wc, clock):
        """Per step, all stream-ordered with no host round trip: fused push
        (emigrants written into the owners' buffers, removed slots listed),
        device-count hole filling, all-reduce of [counts, clock, emigrants]
        (which also orders every sender's writes before the owner reads),
        append of the received records at the device count, and an async
        copy of the reduced vector to pinned memory.

        The host LB bookkeeping (cost vector, efficiency, knapsack / SFC
        attempt, adoption gate, walltime model) runs in order on a worker
        thread while this thread keeps the GPU fed, so even a multi-ms remap
        never stalls the device.  An adoption decided at step s is applied
        physically (owner table + particle migration) before step s + lag on
        every rank -- a deterministic point, so the ranks' collectives stay
        matched.  Ownership never changes a particle's push, and the per-box
        counts are all-reduced over whichever ranks hold the particles, so
        counts, costs, decisions and metrics are exactly those of the
        synchronous loop (tests compare against the oracle)."""
        import os
        import queue

        from .balancer import should_attempt

        cfg, eng, nb = self.cfg, self.engine, self.ba.n_boxes
        lag = max(1, int(os.environ.get("LBX_LB_LAG", "8")))
        adopted, halt = C.c_int32(), C.c_int32()
        work = queue.Queue()
        decided = {}                       # step -> adopted owner table
        st = {"processed": first - 1, "err": None}
        cv = threading.Condition()

        def worker():
            while True:
                item = work.get()
                if item is None:
                    return
                if item[0] == "ratio":             # measured migration price, in step order
                    try:
                        self._set_mig_ratio(item[1])
                    except Exception as e:  # noqa: BLE001
                        st["err"] = e
                    continue
                step, host, ev = item
                try:
                    ev.synchronize()
                    h = host.numpy()
                    k = (2 if clock else 1) * nb
                    if int(h[k + 2]):
                        raise ValueError(f"rank {self.rank}: particles outside the box grid, "
                                         f"staging or receive overflow (code {int(h[k + 2])})")
                    ch = np.ascontiguousarray(h[:nb], dtype=np.int64)
                    kh = np.ascontiguousarray(h[nb:2 * nb]).view(np.uint64) if clock else None
                    _lib.check(_lib.lib.lbx_lb_step(self.lb, step, _lib.ptr(ch), _lib.ptr(kh),
                                                    int(ch.sum()), C.byref(self.souts),
                                                    C.byref(adopted), C.byref(halt)))
                    if adopted.value:
                        owner = np.empty(nb, dtype=np.int64)
                        _lib.check(_lib.lib.lbx_lb_owner(self.lb, _lib.ptr(owner)))
                        decided[step] = owner
                    self.done = step + 1
                    if halt.value:
                        self.halted = True
                except Exception as e:  # noqa: BLE001 -- re-raised on the main thread
                    st["err"] = e
                with cv:
                    st["processed"] = step
                    cv.notify_all()

        def wait_processed(step):
            with cv:
                cv.wait_for(lambda: st["processed"] >= step or st["err"] is not None)
            if st["err"] is not None:
                raise st["err"]

        def apply(d, boundary):
            """Adoption decided at step d, applied before step `boundary`."""
            eng.end_async()                        # host count for the sync migration
            eng.set_owner(decided.pop(d))
            self.moved[d], ratio = self._timed_migration(
                d, lambda: self._migrate_p2p(boundary - 1))
            if ratio is not None:                  # applied before step `boundary`'s LB
                work.put(("ratio", ratio))
            eng.begin_async()

        th = threading.Thread(target=worker, name=f"lbx-lb-rank{self.rank}", daemon=True)
        th.start()
        eng.begin_async()
        try:
            for step in range(first, last):
                if st["err"] is not None:
                    raise st["err"]
                d = step - lag
                if d >= first and should_attempt(self.policy, d, cfg.total_steps):
                    wait_processed(d)
                    if d in decided:
                        apply(d, step)
                if step == cfg.kick.step:
                    eng.kick()
                eng.parity = step & 1
                pev = self._push_events()
                if pev:
                    pev[0].record()
                counts, clk, send_counts, nout = eng.push_async(wp, wc)
                if pev:
                    pev[1].record()
                    self._push_ev = pev
                parts = [counts, clk] if clock else [counts]
                red = torch.cat(parts + [send_counts.sum().reshape(1)])
                self.comm.all_reduce_sum(red)
                eng.unpack_peer_async(step & 1)
                host = torch.empty(red.numel() + 2, dtype=torch.int64, pin_memory=True)
                host.copy_(torch.cat([red, nout]), non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
                work.put((step, host, ev))
            wait_processed(last - 1)
            for d in sorted(decided):              # adoptions of the last `lag` steps
                apply(d, last)
        finally:
            work.put(None)
            th.join()
        eng.end_async()
        return self

    def local_state(self):
        return self.engine.state()

    def result(self) -> RunResult:
        o, cfg, done = self.out, self.cfg, int(self.souts.completed_steps)
        metrics = [StepMetrics(step=s, efficiency_before=float(o["eff_before"][s]),
                               efficiency_after=float(o["eff_after"][s]),
                               adopted=bool(o["adopted"][s]),
                               compute_max=float(o["compute_max"][s]),
                               comm_max=float(o["comm_max"][s]), gather=float(o["gather"][s]),
                               redistribute=float(o["redistribute"][s]),
                               walltime=float(o["walltime"][s]),
                               max_rank_particles=int(o["max_rank_particles"][s]),
                               oom=bool(o["oom"][s])) for s in range(done)]
        na = int(self.souts.n_adoptions)
        eff = np.array([m.efficiency_after for m in metrics])
        summary = {
            "scenario_id": cfg.scenario_id, "n_ranks": cfg.n_ranks,
            "n_boxes": self.ba.n_boxes, "box_grid": list(self.ba.grid_shape),
            "seed": cfg.seed, "policy": policy_kind(self.policy, cfg.total_steps),
            "strategy": self.policy.strategy.value, "interval": self.policy.interval,
            "improvement_threshold": self.policy.improvement_threshold,
            "threshold_mode": self.policy.threshold_mode,
            "static_step": self.policy.static_step, "provider": self.provider.kind,
            "overhead_factor": self.provider.overhead_factor,
            "total_steps": cfg.total_steps, "completed_steps": done,
            "completion_fraction": done / cfg.total_steps,
            "total_walltime": float(sum(m.walltime for m in metrics)),
            "mean_efficiency": float(eff.mean()) if done else 0.0,
            "adoption_count": na, "attempt_count": int(self.souts.n_attempts),
            "oom": bool(done and metrics[-1].oom),
            "final_particles": int(o["n_alive"][done - 1]) if done else self.n_init,
        }
        return RunResult(
            metrics=metrics, summary=summary, cost_trace=o["cost_trace"][:done].copy(),
            initial_owner=self.initial_owner.copy(),
            adoption_snapshots=[(int(o["adopt_steps"][i]), o["adopt_owners"][i].copy())
                                for i in range(na)],
            n_alive=o["n_alive"][:done].copy(),
            count_trace=None if o["count_trace"] is None else o["count_trace"][:done].copy())
