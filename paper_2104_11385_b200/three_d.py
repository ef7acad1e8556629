"""3D box decomposition (config C4: "3D laser-ion acceleration problem, 256
boxes, SFC vs knapsack").  The reference is 2D only, so this is
an extension with PARITY UNPINNED: the 2D rules carried to a third axis and
checked against the oracle's 3D restatement.

Particles: SoA float64 z, y, x, vz, vy, vx in HBM; the fused 3D kernel
(lbx_push_step_3d, 72 B/particle) pushes, absorbs, bins into
(bz*nby + by)*nbx + bx boxes with GpuClock/heuristic costs and compacts
stably; the host step (lbx_lb_step, 3D Morton curve, 3D faces) balances.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .balancer import BalancePolicy, Strategy
from .cost import CostProvider
from .device import Context, _stream, require_cuda
from .errors import ConfigError


@dataclass(frozen=True)
class Scenario3D:
    scenario_id: str
    domain_extent: tuple[int, int, int]      # (Nz, Ny, Nx) cells
    box_size: int
    n_ranks: int
    center: tuple[float, float, float]
    core_radius: float
    edge_scale: float
    particles_per_cell: float
    kick_step: int
    kick_speed: float
    kick_drift: float
    total_steps: int
    work_weights: tuple[float, float] = (0.75, 0.25)
    initial_mapping: str = "slab"
    seed: int = 1

    def __post_init__(self):
        if len(self.domain_extent) != 3 or any(e % self.box_size for e in self.domain_extent):
            raise ConfigError("3D extent must be three multiples of box_size")
        if self.box_size & (self.box_size - 1):
            raise ConfigError("3D box_size must be a power of two")

    @property
    def grid(self):
        return tuple(e // self.box_size for e in self.domain_extent)

    @property
    def n_boxes(self):
        g = self.grid
        return g[0] * g[1] * g[2]


def sample_blob_3d(cfg: Scenario3D) -> np.ndarray:
    """Spherical blob: uniform core, exponential skirt; every cell within
    core + 12*scale + 1 contributes floor(ppc) (+ Bernoulli) candidates,
    uniform in the cell, accepted with exp(-(rho - core)/scale) outside the
    core.  PCG64 stream (seed, 1)."""
    nz, ny, nx = cfg.domain_extent
    c = np.array(cfg.center)
    reach = cfg.core_radius + 12.0 * cfg.edge_scale + 1.0
    lo = np.maximum(np.floor(c - reach).astype(int), 0)
    hi = np.minimum(np.ceil(c + reach).astype(int), [nz, ny, nx])
    g = np.stack(np.meshgrid(*[np.arange(lo[a], hi[a]) for a in range(3)], indexing="ij"),
                 -1).reshape(-1, 3)
    g = g[np.sqrt(((g + 0.5 - c) ** 2).sum(1)) <= reach]
    rng = np.random.default_rng((int(cfg.seed), 1))
    whole = int(math.floor(cfg.particles_per_cell))
    per = np.full(len(g), whole, dtype=np.int64)
    frac = cfg.particles_per_cell - whole
    if frac > 0:
        per += rng.random(len(g)) < frac
    pos = np.repeat(g, per, axis=0).astype(np.float64) + rng.random((int(per.sum()), 3))
    rho = np.sqrt(((pos - c) ** 2).sum(1))
    if cfg.edge_scale > 0:
        acc = np.where(rho <= cfg.core_radius, 1.0,
                       np.exp(-(rho - cfg.core_radius) / cfg.edge_scale))
    else:
        acc = (rho <= cfg.core_radius).astype(np.float64)
    return np.ascontiguousarray(pos[rng.random(len(pos)) < acc])


def kick_velocities_3d(pos: np.ndarray, cfg: Scenario3D) -> np.ndarray:
    rng = np.random.default_rng((int(cfg.seed), 2))
    f = rng.uniform(0.5, 1.5, size=len(pos))
    d = pos - np.array(cfg.center)
    rho = np.sqrt((d ** 2).sum(1))
    u = np.divide(d, rho[:, None], out=np.zeros_like(d), where=rho[:, None] > 0)
    v = (cfg.kick_speed * f)[:, None] * u
    v[:, 0] += cfg.kick_drift
    return np.ascontiguousarray(v)


class Simulation3D:
    """Device-resident 3D run: fused 3D kernel per step + host LB step."""

    def __init__(self, cfg: Scenario3D, policy: BalancePolicy, provider: CostProvider, *,
                 device="cuda:0", positions=None, kick=None, record_counts=False,
                 stable_order=True):
        """stable_order=False compacts absorbed particles by O(removed) hole
        filling (particle order then differs from the sequential rule)."""
        from .balancer import knapsack_assign, sfc_assign
        from .cost import CostVector
        from .decomposition import morton_order_3d

        if provider.device_kind not in (0, 1, 2, 3):
            raise ConfigError(f"provider {provider.kind!r} not supported in 3D")
        self.cfg, self.policy, self.provider = cfg, policy, provider
        self.dev = require_cuda(device)
        pos = sample_blob_3d(cfg) if positions is None else positions
        n = self.n_init = int(pos.shape[0])
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.arr = {k: torch.zeros(n + 2, **f64) for k in ("z", "y", "x", "vz", "vy", "vx")}
        pt = torch.as_tensor(pos).to(self.dev)
        for a, k in enumerate(("z", "y", "x")):
            self.arr[k][:n].copy_(pt[:, a])
        self.kick = None
        if cfg.kick_step < cfg.total_steps:
            kv = kick if kick is not None else kick_velocities_3d(np.asarray(pos), cfg)
            self.kick = torch.as_tensor(kv).to(self.dev)
        self.ctx = Context(self.dev, capacity=n)
        self.ctx.set_count(n)
        M = cfg.box_size
        gz, gy, gx = cfg.grid
        ids = ((torch.div(pt[:, 0], M, rounding_mode="trunc").long() * gy
                + torch.div(pt[:, 1], M, rounding_mode="trunc").long()) * gx
               + torch.div(pt[:, 2], M, rounding_mode="trunc").long())
        counts0 = torch.bincount(ids, minlength=cfg.n_boxes).cpu().numpy()
        work0 = cfg.work_weights[0] * counts0.astype(np.float64) + cfg.work_weights[1] * M ** 3
        if cfg.initial_mapping == "slab":
            own = np.empty(cfg.n_boxes, dtype=np.int64)
            _lib.check(_lib.lib.lbx_slab_mapping(cfg.n_boxes, cfg.n_ranks, _lib.ptr(own)))
        elif cfg.initial_mapping == "knapsack":
            own = knapsack_assign(CostVector(values=work0), cfg.n_ranks).owner
        else:
            own = sfc_assign(CostVector(values=work0), morton_order_3d(cfg.grid), cfg.n_ranks).owner
        self.initial_owner = np.array(own, dtype=np.int64)
        w = getattr(provider, "weights", None)
        mc = getattr(provider, "cfg", None)
        self.wp, self.wc = (w.w_particle, w.w_cell) if w else (0.75, 0.25)
        conf = _lib.SimConfig(
            extent_z=cfg.domain_extent[0], extent_x=cfg.domain_extent[2], box_size=M,
            n_ranks=cfg.n_ranks, total_steps=cfg.total_steps, kick_step=cfg.kick_step,
            strategy=0 if policy.strategy is Strategy.KNAPSACK else 1, interval=policy.interval,
            improvement_threshold=policy.improvement_threshold,
            threshold_relative=1 if policy.threshold_mode == "relative" else 0,
            cap_factor=policy.knapsack_cap_factor,
            static_step=-1 if policy.static_step is None else policy.static_step,
            cost_kind=provider.device_kind, w_particle=self.wp, w_cell=self.wc,
            noise_amplitude=mc.noise_amplitude if mc else 0.0, noise_seed=mc.seed if mc else 0,
            overhead_factor=provider.overhead_factor, work_wp=cfg.work_weights[0],
            work_wc=cfg.work_weights[1], comm_per_face=0.0, gather=0.0,
            redistribute_per_particle=0.0, redistribute_latency=0.0, capacity_particles=-1,
            physics=0, pic_dt=0.5, pic_q_over_m=-1.0, pic_q_times_w=-1e-4,
            extent_y=cfg.domain_extent[1], migration_ratio=policy.migration_ratio,
            clock_mode=getattr(provider, "clock_mode", 0))
        self.conf = conf
        h = C.c_void_p()
        _lib.check(_lib.lib.lbx_lb_create(C.byref(h), C.byref(conf), _lib.ptr(self.initial_owner)))
        self.lb = h
        T, nb = cfg.total_steps, cfg.n_boxes
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
        self.out = o
        self.souts = _lib.SimOutputs(
            *(_lib.ptr(o.get(k)) for k in ("eff_before", "eff_after", "adopted", "attempted",
                                           "compute_max", "comm_max", "gather", "redistribute",
                                           "walltime", "max_rank_particles", "oom", "n_alive",
                                           "cost_trace", "count_trace", "clock_trace", "owner",
                                           "adopt_steps", "adopt_owners")), None, 0, 0, 0)
        self.dcounts = torch.zeros(nb, dtype=torch.int64, device=self.dev)
        self.dcost = torch.zeros(nb, **f64)
        self.dclk = torch.zeros(nb, dtype=torch.int64, device=self.dev)
        self.dn = torch.zeros(2, dtype=torch.int64, device=self.dev)
        self.n = n
        self.done = 0
        self.kernel_ms = []
        self.stable_order = stable_order
        self.removed = None if stable_order else torch.empty(n + 2, dtype=torch.int64,
                                                             device=self.dev)

    def close(self):
        if getattr(self, "lb", None):
            _lib.lib.lbx_lb_destroy(self.lb)
            self.lb = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step_device(self):
        """Enqueue one fused 3D step (no host sync)."""
        a = self.arr
        c = self.cfg
        args = _lib.Step3DArgs(
            *(_lib.ptr(a[k]) for k in ("z", "y", "x", "vz", "vy", "vx")),
            c.domain_extent[0], c.domain_extent[1], c.domain_extent[2], c.box_size,
            float(self.wp), float(self.wc),
            _lib.LBX_STEP_CLOCK if self.provider.device_kind == 3 else 0,
            _lib.ptr(self.dcounts), _lib.ptr(self.dcost), _lib.ptr(self.dclk),
            _lib.ptr(self.dn), _lib.ptr(self.dn[1:]), _lib.ptr(self.removed),
            0 if self.removed is None else self.removed.numel())
        self.ctx.set_count(self.n)
        _lib.check(_lib.lib.lbx_push_step_3d(self.ctx.handle, C.byref(args), _stream(self.dev)))

    def run(self, first=None, last=None):
        first = self.done if first is None else first
        last = self.cfg.total_steps if last is None else last
        adopted, halt = C.c_int32(), C.c_int32()
        clock = self.provider.device_kind == 3
        for step in range(first, last):
            if step == self.cfg.kick_step and self.kick is not None:
                n = self.n
                for col, k in enumerate(("vz", "vy", "vx")):
                    self.arr[k][:n].copy_(self.kick[:n, col])
                self.kick = None
            self.step_device()
            h = torch.cat([self.dn, self.dcounts, self.dclk]).cpu().numpy()
            if h[1]:
                raise ValueError(f"{int(h[1])} particles outside the box grid")
            if not self.stable_order:
                a = self.arr
                _lib.check(_lib.lib.lbx_fill_holes(
                    self.ctx.handle, *(_lib.ptr(a[k]) for k in ("z", "x", "y", "vz", "vy", "vx")),
                    _lib.ptr(self.removed), self.n - int(h[0]), int(h[0]), _stream(self.dev)))
            self.n = int(h[0])
            nb = self.cfg.n_boxes
            counts = np.ascontiguousarray(h[2:2 + nb])
            clk = np.ascontiguousarray(h[2 + nb:2 + 2 * nb]).view(np.uint64) if clock else None
            _lib.check(_lib.lib.lbx_lb_step(self.lb, step, _lib.ptr(counts), _lib.ptr(clk), self.n,
                                            C.byref(self.souts), C.byref(adopted), C.byref(halt)))
            self.done = step + 1
        return self

    def owner_at(self, step):
        own = self.initial_owner.copy()
        for i in range(int(self.souts.n_adoptions)):
            if self.out["adopt_steps"][i] <= step:
                own = self.out["adopt_owners"][i].copy()
        return own

    def state(self):
        n = self.n
        pos = torch.stack([self.arr[k][:n] for k in ("z", "y", "x")], 1).cpu().numpy()
        vel = torch.stack([self.arr[k][:n] for k in ("vz", "vy", "vx")], 1).cpu().numpy()
        return pos, vel


# ---------------------------------------------------------------------------
# Multi-GPU 3D (config C4 strong scaling): one rank per GPU owns the particles
# of its boxes; the 3D analogue of parallel.DistributedSimulation (its
# communicators, non-fused exchange).
# ---------------------------------------------------------------------------

REC3 = 6   # (z, y, x, vz, vy, vx)


def box_ids_3d(pos: np.ndarray, cfg: Scenario3D) -> np.ndarray:
    g = cfg.grid
    b = np.trunc(np.asarray(pos) / cfg.box_size).astype(np.int64)
    return (b[:, 0] * g[1] + b[:, 1]) * g[2] + b[:, 2]


def initial_owner_3d(cfg: Scenario3D, pos: np.ndarray) -> np.ndarray:
    """Simulation3D's initial mapping: slab, or knapsack / SFC of true work."""
    from .balancer import knapsack_assign, sfc_assign
    from .cost import CostVector
    from .decomposition import morton_order_3d

    counts0 = np.bincount(box_ids_3d(pos, cfg), minlength=cfg.n_boxes)
    work0 = cfg.work_weights[0] * counts0.astype(np.float64) + cfg.work_weights[1] * cfg.box_size ** 3
    if cfg.initial_mapping == "slab":
        own = np.empty(cfg.n_boxes, dtype=np.int64)
        _lib.check(_lib.lib.lbx_slab_mapping(cfg.n_boxes, cfg.n_ranks, _lib.ptr(own)))
        return own
    if cfg.initial_mapping == "knapsack":
        return np.asarray(knapsack_assign(CostVector(values=work0), cfg.n_ranks).owner)
    return np.asarray(sfc_assign(CostVector(values=work0), morton_order_3d(cfg.grid),
                                 cfg.n_ranks).owner)


def lb_config_3d(cfg: Scenario3D, policy: BalancePolicy, provider: CostProvider):
    w = getattr(provider, "weights", None)
    mc = getattr(provider, "cfg", None)
    wp, wc = (w.w_particle, w.w_cell) if w else (0.75, 0.25)
    conf = _lib.SimConfig(
        extent_z=cfg.domain_extent[0], extent_x=cfg.domain_extent[2], box_size=cfg.box_size,
        n_ranks=cfg.n_ranks, total_steps=cfg.total_steps, kick_step=cfg.kick_step,
        strategy=0 if policy.strategy is Strategy.KNAPSACK else 1, interval=policy.interval,
        improvement_threshold=policy.improvement_threshold,
        threshold_relative=1 if policy.threshold_mode == "relative" else 0,
        cap_factor=policy.knapsack_cap_factor,
        static_step=-1 if policy.static_step is None else policy.static_step,
        cost_kind=provider.device_kind, w_particle=wp, w_cell=wc,
        noise_amplitude=mc.noise_amplitude if mc else 0.0, noise_seed=mc.seed if mc else 0,
        overhead_factor=provider.overhead_factor, work_wp=cfg.work_weights[0],
        work_wc=cfg.work_weights[1], comm_per_face=0.0, gather=0.0,
        redistribute_per_particle=0.0, redistribute_latency=0.0, capacity_particles=-1,
        physics=0, pic_dt=0.5, pic_q_over_m=-1.0, pic_q_times_w=-1e-4,
        extent_y=cfg.domain_extent[1], migration_ratio=policy.migration_ratio,
        clock_mode=getattr(provider, "clock_mode", 0))
    return conf, wp, wc


class Engine3D:
    """This rank's 3D particles in HBM and the libLBX 3D exchange kernels
    (lbx_push_step_3d_exchange / lbx_partition_3d, lbx_group_by_dest,
    lbx_unpack, lbx_fill_holes with z, y, x, vz, vy, vx in the six slots).
    Before the kick the pushes read a zero velocity buffer and the velocity
    arrays hold the pending kick velocities, so migration carries them."""

    def __init__(self, cfg: Scenario3D, rank, world, device, pos, kick, capacity, clock):
        self.dev = require_cuda(device)
        self.cfg, self.rank, self.world, self.clock = cfg, rank, world, clock
        cap = int(capacity) + 2
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.a = {k: torch.zeros(cap, **f64) for k in ("z", "y", "x", "vz", "vy", "vx")}
        n = int(pos.shape[0])
        p = torch.as_tensor(np.asarray(pos)).to(self.dev)
        for c, k in enumerate(("z", "y", "x")):
            self.a[k][:n].copy_(p[:, c])
        self.kicked = kick is None
        if kick is not None:
            kv = torch.as_tensor(np.asarray(kick)).to(self.dev)
            for c, k in enumerate(("vz", "vy", "vx")):
                self.a[k][:n].copy_(kv[:, c])
        self.zero_v = torch.zeros(cap, **f64)
        self.n, self.capacity = n, int(capacity)
        self.stage = torch.empty((cap, REC3), **f64)
        self.stage_dest = torch.empty(cap, dtype=torch.int32, device=self.dev)
        self.removed = torch.empty(cap, dtype=torch.int64, device=self.dev)
        self.send_counts = torch.zeros(world, dtype=torch.int64, device=self.dev)
        self.owner = torch.zeros(cfg.n_boxes, dtype=torch.int32, device=self.dev)
        nb = cfg.n_boxes
        self.counts = torch.zeros(nb, dtype=torch.int64, device=self.dev)
        self.cost = torch.zeros(nb, **f64)
        self.clk = torch.zeros(nb, dtype=torch.int64, device=self.dev)
        self.nout = torch.zeros(2, dtype=torch.int64, device=self.dev)
        self.ctx = Context(self.dev, capacity=cap)
        self.launches = 0

    def _ptrs(self):
        return [_lib.ptr(self.a[k]) for k in ("z", "y", "x", "vz", "vy", "vx")]

    def _ex(self):
        return _lib.ExchangeArgs(
            _lib.ptr(self.owner), self.rank, self.world, _lib.ptr(self.stage),
            _lib.ptr(self.stage_dest), self.capacity + 2, _lib.ptr(self.send_counts),
            None, None, _lib.ptr(self.removed), self.capacity + 2)

    def set_owner(self, owner: np.ndarray):
        self.owner.copy_(torch.from_numpy(np.asarray(owner, dtype=np.int32)))

    def kick(self):
        self.kicked = True

    def push(self, wp, wc):
        c = self.cfg
        self.send_counts.zero_()
        self.ctx.set_count(self.n)
        p = self._ptrs()
        v = p[3:] if self.kicked else [_lib.ptr(self.zero_v)] * 3
        args = _lib.Step3DArgs(
            *p[:3], *v, c.domain_extent[0], c.domain_extent[1], c.domain_extent[2], c.box_size,
            float(wp), float(wc), _lib.LBX_STEP_CLOCK if self.clock else 0,
            _lib.ptr(self.counts), _lib.ptr(self.cost), _lib.ptr(self.clk),
            _lib.ptr(self.nout), _lib.ptr(self.nout[1:]), None, 0)
        ex = self._ex()
        _lib.check(_lib.lib.lbx_push_step_3d_exchange(self.ctx.handle, C.byref(args), C.byref(ex),
                                                      _stream(self.dev)))
        self.launches += 2   # set_count, fused 3D step
        return self.counts, self.clk, self.send_counts, self.nout

    def partition(self):
        c = self.cfg
        self.send_counts.zero_()
        self.ctx.set_count(self.n)
        ex = self._ex()
        _lib.check(_lib.lib.lbx_partition_3d(
            self.ctx.handle, *self._ptrs(), c.domain_extent[0], c.domain_extent[1],
            c.domain_extent[2], c.box_size, C.byref(ex), _lib.ptr(self.nout), _stream(self.dev)))
        self.launches += 3
        return self.send_counts, self.nout

    def commit(self, nout_host):
        if int(nout_host[1]) != 0:
            raise ValueError("particles outside the box grid or staging overflow "
                             f"(code {int(nout_host[1])})")
        n_new = int(nout_host[0])
        _lib.check(_lib.lib.lbx_fill_holes(self.ctx.handle, *self._ptrs(), _lib.ptr(self.removed),
                                           self.n - n_new, n_new, _stream(self.dev)))
        self.launches += 3
        self.n = n_new

    def pack(self, sc: list) -> torch.Tensor:
        total = int(sum(sc))
        send = torch.empty((total, REC3), dtype=torch.float64, device=self.dev)
        if total:
            cur = torch.tensor(np.concatenate(([0], np.cumsum(sc)[:-1])), dtype=torch.int64,
                               device=self.dev)
            _lib.check(_lib.lib.lbx_group_by_dest(_lib.ptr(self.stage), _lib.ptr(self.stage_dest),
                                                  total, self.world, _lib.ptr(cur), _lib.ptr(send),
                                                  _stream(self.dev)))
            self.launches += 1
        return send

    def unpack(self, recv: torch.Tensor):
        m = int(recv.shape[0])
        if self.n + m > self.capacity:
            raise MemoryError(f"rank {self.rank}: {self.n + m} particles exceed capacity "
                              f"{self.capacity}")
        if m:
            recv = recv.contiguous()
            _lib.check(_lib.lib.lbx_unpack(_lib.ptr(recv), m, self.n, *self._ptrs(),
                                           _stream(self.dev)))
            self.launches += 1
        self.n += m

    def state(self):
        n = self.n
        pos = torch.stack([self.a[k][:n] for k in ("z", "y", "x")], 1).cpu().numpy()
        vel = torch.stack([self.a[k][:n] for k in ("vz", "vy", "vx")], 1).cpu().numpy()
        if not self.kicked:
            vel = np.zeros_like(vel)
        return pos, vel


class Distributed3D:
    """Config C4 on `world` ranks: rank r holds the particles of the boxes
    it owns; every step the fused 3D kernel pushes them, counts the
    survivors per box and stages those now in another rank's boxes; one
    all-reduce of [counts, clock, emigrants] makes the cost vector global,
    the records move in one all-to-all, and every rank runs the same host LB
    step (lbx_lb_step: 3D Morton curve, 3D faces), so all ranks adopt the
    same mappings; an adoption migrates the re-owned boxes' particles.
    Results equal Simulation3D's (counts, costs, mappings; the particle
    multiset -- local order is not kept).  Kick: the scenario's velocities
    are zero before cfg.kick_step (Simulation3D's rule)."""

    def __init__(self, cfg: Scenario3D, policy: BalancePolicy, provider: CostProvider, *,
                 comm=None, engine_factory=None, device="cuda:0", positions=None, kick=None,
                 replicas: int = 1, capacity=None, record_counts=False):
        from .parallel import TorchComm

        if provider.device_kind not in (0, 1, 2, 3):
            raise ConfigError(f"provider {provider.kind!r} not supported in 3D")
        self.comm = comm or TorchComm()
        self.rank, self.world = self.comm.rank, self.comm.world
        if cfg.n_ranks != self.world:
            raise ConfigError(f"scenario has {cfg.n_ranks} ranks, communicator {self.world}")
        self.cfg, self.policy, self.provider = cfg, policy, provider
        pos = sample_blob_3d(cfg) if positions is None else np.asarray(positions)
        kv = None
        if cfg.kick_step < cfg.total_steps:
            kv = kick_velocities_3d(pos, cfg) if kick is None else np.asarray(kick)
        self.initial_owner = initial_owner_3d(cfg, pos)
        mine = self.initial_owner[box_ids_3d(pos, cfg)] == self.rank
        local = np.tile(pos[mine], (replicas, 1))
        klocal = None if kv is None else np.tile(kv[mine], (replicas, 1))
        self.n_total = pos.shape[0] * replicas
        cap = capacity if capacity is not None else self.n_total
        factory = engine_factory or Engine3D
        self.engine = factory(cfg, self.rank, self.world, device, local, klocal, cap,
                              provider.device_kind == 3)
        self.engine.set_owner(self.initial_owner)
        self.conf, self.wp, self.wc = lb_config_3d(cfg, policy, provider)
        h = C.c_void_p()
        own = np.ascontiguousarray(self.initial_owner, dtype=np.int64)
        _lib.check(_lib.lib.lbx_lb_create(C.byref(h), C.byref(self.conf), _lib.ptr(own)))
        self.lb = h
        T, nb = cfg.total_steps, cfg.n_boxes
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
        self.out = o
        self.souts = _lib.SimOutputs(
            *(_lib.ptr(o.get(k)) for k in ("eff_before", "eff_after", "adopted", "attempted",
                                           "compute_max", "comm_max", "gather", "redistribute",
                                           "walltime", "max_rank_particles", "oom", "n_alive",
                                           "cost_trace", "count_trace", "clock_trace", "owner",
                                           "adopt_steps", "adopt_owners")), None, 0, 0, 0)
        self.moved = np.zeros(T, dtype=np.int64)
        self.emigrated = np.zeros(T, dtype=np.int64)
        self.done = 0

    def close(self):
        if getattr(self, "lb", None):
            _lib.lib.lbx_lb_destroy(self.lb)
            self.lb = None

    def _records(self, send_counts, nout):
        """Counts all-to-all, one host copy, commit, record all-to-all."""
        recv_counts = self.comm.exchange_counts(send_counts)
        h = torch.cat([nout, send_counts, recv_counts]).cpu().numpy()
        self.engine.commit(h[:2])
        w = self.world
        sc, rc = [int(v) for v in h[2:2 + w]], [int(v) for v in h[2 + w:2 + 2 * w]]
        if sum(sc) or sum(rc):
            send = self.engine.pack(sc)
            self.engine.unpack(self.comm.exchange_records(send, sc, rc))
        return sum(sc)

    def run(self, first=None, last=None):
        cfg = self.cfg
        first = self.done if first is None else first
        last = cfg.total_steps if last is None else last
        clock = self.provider.device_kind == 3
        nb = cfg.n_boxes
        adopted, halt = C.c_int32(), C.c_int32()
        for step in range(first, last):
            if step == cfg.kick_step:
                self.engine.kick()
            counts, clk, send_counts, nout = self.engine.push(self.wp, self.wc)
            parts = [counts, clk] if clock else [counts]
            red = torch.cat(parts + [send_counts.sum().reshape(1)])
            self.comm.all_reduce_sum(red)      # global per-box counts / clock tally
            h = red.cpu().numpy()
            ch = np.ascontiguousarray(h[:nb], dtype=np.int64)
            kh = np.ascontiguousarray(h[nb:2 * nb]).view(np.uint64) if clock else None
            self.emigrated[step] = int(h[-1])
            if int(h[-1]):
                self._records(send_counts, nout)
            else:
                self.engine.commit(nout.cpu().numpy())
            _lib.check(_lib.lib.lbx_lb_step(self.lb, step, _lib.ptr(ch), _lib.ptr(kh),
                                            int(ch.sum()), C.byref(self.souts),
                                            C.byref(adopted), C.byref(halt)))
            if adopted.value:
                owner = np.empty(nb, dtype=np.int64)
                _lib.check(_lib.lib.lbx_lb_owner(self.lb, _lib.ptr(owner)))
                self.engine.set_owner(owner)
                send_counts, nout = self.engine.partition()
                self.moved[step] = self._records(send_counts, nout)
            self.done = step + 1
        return self

    def owner_at(self, step):
        own = self.initial_owner.copy()
        for i in range(int(self.souts.n_adoptions)):
            if self.out["adopt_steps"][i] <= step:
                own = self.out["adopt_owners"][i].copy()
        return own

    def local_state(self):
        return self.engine.state()
