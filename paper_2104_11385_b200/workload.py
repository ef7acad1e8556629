"""Scenario model and the stepping loop -- API mirror of lbsim/workload.py.

Scenario construction (blob sampling, kick velocities) is host-side numpy
with the reference's exact PCG64 streams, as in the reference; everything
per step runs in libLBX: the fused sm_100a step kernel and the native C++
loop (``lbx_sim_run``) that assesses costs, balances and prices each step.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from . import _lib
from .balancer import BalanceOutcome, BalancePolicy, Strategy
from .cost import CostProvider, CostVector
from .decomposition import (BoxArray, DistributionMapping, build_box_array,
                            morton_order, round_robin_mapping, slab_mapping)
from .errors import ConfigError

SKIRT_CUTOFF = 12.0      # acceptance below exp(-12) treated as zero (workload.py:34)
STREAM_INIT, STREAM_KICK = 1, 2


@dataclass(frozen=True)
class BlobSpec:
    center: tuple[float, float]
    core_radius: float
    edge_scale: float
    particles_per_cell: float

    def __post_init__(self):
        object.__setattr__(self, "center", tuple(self.center))
        if self.core_radius < 0 or self.edge_scale < 0:
            raise ConfigError("blob radii must be nonnegative")
        if self.particles_per_cell < 0:
            raise ConfigError("blob particles_per_cell must be nonnegative")


@dataclass(frozen=True)
class KickSpec:
    step: int
    speed: float
    drift: float = 0.0

    def __post_init__(self):
        if self.step < 0:
            raise ConfigError("kick step must be nonnegative")
        if self.speed < 0:
            raise ConfigError("kick speed must be nonnegative")


@dataclass(frozen=True)
class CostModel:
    comm_per_face: float
    gather: float
    redistribute_per_particle: float
    redistribute_latency: float

    def __post_init__(self):
        for k in ("comm_per_face", "gather", "redistribute_per_particle",
                  "redistribute_latency"):
            if getattr(self, k) < 0:
                raise ConfigError(f"cost model field {k} must be >= 0")


@dataclass(frozen=True)
class ScenarioConfig:
    scenario_id: str
    domain_extent: tuple[int, int]
    box_size: int
    n_ranks: int
    blob: BlobSpec
    kick: KickSpec
    total_steps: int
    compute_fraction: float = 0.5
    work_weights: tuple[float, float] = (0.75, 0.25)
    costs: CostModel | None = None
    capacity_particles: int | None = None
    initial_mapping: str = "slab"
    seed: int = 1

    def __post_init__(self):
        object.__setattr__(self, "domain_extent", tuple(self.domain_extent))
        object.__setattr__(self, "work_weights", tuple(self.work_weights))
        if self.total_steps < 1:
            raise ConfigError("total_steps must be >= 1")
        if not 0.0 < self.compute_fraction <= 1.0:
            raise ConfigError("compute_fraction must be in (0, 1]")
        if self.n_ranks < 1:
            raise ConfigError("n_ranks must be >= 1")
        if min(self.work_weights) < 0:
            raise ConfigError("work weights must be nonnegative")
        if self.initial_mapping not in ("slab", "roundrobin", "knapsack", "sfc"):
            raise ConfigError("initial_mapping must be slab, roundrobin, knapsack, or sfc; "
                              f"got {self.initial_mapping!r}")
        if self.capacity_particles is not None and self.capacity_particles < 1:
            raise ConfigError("capacity_particles must be >= 1 when set")


@dataclass(frozen=True)
class WorkloadState:
    """Host snapshot of the particle ensemble (workload.py:128-145)."""

    positions: np.ndarray
    velocities: np.ndarray
    step: int
    per_box_particles: np.ndarray

    def __post_init__(self):
        for k in ("positions", "velocities", "per_box_particles"):
            a = np.array(getattr(self, k), copy=True)
            a.flags.writeable = False
            object.__setattr__(self, k, a)

    @property
    def n_particles(self) -> int:
        return int(self.positions.shape[0])


@dataclass(frozen=True)
class StepMetrics:
    step: int
    efficiency_before: float
    efficiency_after: float
    adopted: bool
    compute_max: float
    comm_max: float
    gather: float
    redistribute: float
    walltime: float
    max_rank_particles: int
    oom: bool


@dataclass
class RunResult:
    metrics: list[StepMetrics]
    summary: dict
    cost_trace: np.ndarray
    initial_owner: np.ndarray
    adoption_snapshots: list[tuple[int, np.ndarray]]
    # B200 extras: per-step survivors, counts / clock tallies when recorded,
    # per-step fused-kernel milliseconds, final particle state.
    n_alive: np.ndarray | None = None
    count_trace: np.ndarray | None = None
    clock_trace: np.ndarray | None = None
    kernel_ms: np.ndarray | None = None
    final_state: object = field(default=None, repr=False)


def box_array_for(cfg: ScenarioConfig) -> BoxArray:
    return build_box_array(cfg.domain_extent, cfg.box_size)


@lru_cache(maxsize=64)
def resolve_costs(cfg: ScenarioConfig) -> CostModel:
    """Walltime-model coefficients, derived from geometry when not given
    (workload.py:180-215): comm ~ compute*(1-f)/f near balance, one gather
    = 2.5% of a balanced step, moving every particle = 3 steps + 5% latency."""
    if cfg.costs is not None:
        return cfg.costs
    nz, nx = cfg.domain_extent
    r, s = cfg.blob.core_radius, cfg.blob.edge_scale
    est_p = cfg.blob.particles_per_cell * (math.pi * r * r + 2.0 * math.pi * r * s)
    wp, wc = cfg.work_weights
    c_avg = (wp * est_p + wc * (nz * nx)) / cfg.n_ranks
    w_est = c_avg / cfg.compute_fraction
    nbz, nbx = nz // cfg.box_size, nx // cfg.box_size
    faces = 2 * nbz * nbx - nbz - nbx
    per_rank = max(2.0 * faces / cfg.n_ranks * (1.0 - 1.0 / cfg.n_ranks), 1.0)
    comm = c_avg * (1.0 - cfg.compute_fraction) / cfg.compute_fraction
    return CostModel(comm_per_face=comm / per_rank, gather=0.025 * w_est,
                     redistribute_per_particle=3.0 * w_est / max(est_p, 1.0),
                     redistribute_latency=0.05 * w_est)


def sample_blob(cfg: ScenarioConfig) -> np.ndarray:
    """Initial positions [n, 2] (workload.py:218-265): every cell whose centre
    is within core + 12*scale + 1 contributes floor(ppc) candidates (+1 with
    probability frac(ppc)), uniform in the cell; a candidate at radius rho
    is kept with probability 1 in the core, exp(-(rho-core)/scale) outside.
    PCG64 stream (seed, 1), draws in the reference's order."""
    nz, nx = cfg.domain_extent
    b = cfg.blob
    reach = b.core_radius + SKIRT_CUTOFF * b.edge_scale + 1.0
    cz = np.repeat(np.arange(nz), nx)
    cx = np.tile(np.arange(nx), nz)
    sel = np.hypot(cz + 0.5 - b.center[0], cx + 0.5 - b.center[1]) <= reach
    cz, cx = cz[sel], cx[sel]
    if cz.size == 0 or b.particles_per_cell == 0:
        raise ConfigError("scenario produces zero particles; check blob radius and "
                          "particles_per_cell")
    rng = np.random.default_rng((int(cfg.seed), STREAM_INIT))
    whole = int(math.floor(b.particles_per_cell))
    frac = b.particles_per_cell - whole
    per_cell = np.full(cz.size, whole, dtype=np.int64)
    if frac > 0.0:
        per_cell += rng.random(cz.size) < frac
    total = int(per_cell.sum())
    if total == 0:
        raise ConfigError("scenario produces zero particles; check blob radius and "
                          "particles_per_cell")
    jitter = rng.random((total, 2))
    pos = np.empty((total, 2))
    pos[:, 0] = np.repeat(cz, per_cell).astype(np.float64) + jitter[:, 0]
    pos[:, 1] = np.repeat(cx, per_cell).astype(np.float64) + jitter[:, 1]
    rho = np.hypot(pos[:, 0] - b.center[0], pos[:, 1] - b.center[1])
    if b.edge_scale > 0.0:
        p_keep = np.where(rho <= b.core_radius, 1.0,
                          np.exp(-(rho - b.core_radius) / b.edge_scale))
    else:
        p_keep = (rho <= b.core_radius).astype(np.float64)
    pos = np.ascontiguousarray(pos[rng.random(total) < p_keep])
    if pos.shape[0] == 0:
        raise ConfigError("scenario produces zero particles; check blob radius and "
                          "particles_per_cell")
    return pos


def kick_velocities(positions: np.ndarray, cfg: ScenarioConfig) -> np.ndarray:
    """Radial kick speed*U(0.5,1.5)*r_hat + (drift, 0), PCG64 stream
    (seed, 2) in particle order (workload.py:272-283)."""
    rng = np.random.default_rng((int(cfg.seed), STREAM_KICK))
    f = rng.uniform(0.5, 1.5, size=positions.shape[0])
    dz = positions[:, 0] - cfg.blob.center[0]
    dx = positions[:, 1] - cfg.blob.center[1]
    rho = np.hypot(dz, dx)
    uz = np.divide(dz, rho, out=np.zeros_like(dz), where=rho > 0)
    ux = np.divide(dx, rho, out=np.zeros_like(dx), where=rho > 0)
    sp = cfg.kick.speed * f
    out = np.empty_like(positions)
    out[:, 0] = sp * uz + cfg.kick.drift
    out[:, 1] = sp * ux
    return out


def init_scenario(cfg: ScenarioConfig) -> WorkloadState:
    """Sampled blob + device-binned counts, velocities zero."""
    from . import kernels

    pos = sample_blob(cfg)
    nbz, nbx = cfg.domain_extent[0] // cfg.box_size, cfg.domain_extent[1] // cfg.box_size
    counts = kernels.bin_particles(pos, float(cfg.box_size), nbz, nbx)
    return WorkloadState(positions=pos, velocities=np.zeros_like(pos), step=0,
                         per_box_particles=counts)


def advance(state: WorkloadState, cfg: ScenarioConfig) -> WorkloadState:
    """One host-visible step through the drop-in kernels (workload.py:286-300)."""
    from . import kernels

    if state.step >= cfg.total_steps:
        raise ValueError(f"cannot advance past total_steps={cfg.total_steps}")
    vel = kick_velocities(state.positions, cfg) if state.step == cfg.kick.step \
        else state.velocities
    pos, vel = kernels.advance_particles(state.positions, vel, float(cfg.domain_extent[0]),
                                         float(cfg.domain_extent[1]))
    nbz, nbx = cfg.domain_extent[0] // cfg.box_size, cfg.domain_extent[1] // cfg.box_size
    counts = kernels.bin_particles(pos, float(cfg.box_size), nbz, nbx)
    return WorkloadState(positions=pos, velocities=vel, step=state.step + 1,
                         per_box_particles=counts)


def true_work(state_or_counts, cfg: ScenarioConfig) -> np.ndarray:
    """Ground-truth per-box work w_p*count + w_c*M^2 (workload.py:303-311)."""
    counts = getattr(state_or_counts, "per_box_particles", state_or_counts)
    wp, wc = cfg.work_weights
    return wp * np.asarray(counts).astype(np.float64) + wc * float(cfg.box_size ** 2)


def step_walltime(rank_compute, dm: DistributionMapping, ba: BoxArray,
                  outcome: BalanceOutcome, prev_dm: DistributionMapping,
                  state: WorkloadState, cfg: ScenarioConfig, *, overhead: float = 1.0,
                  faces=None) -> StepMetrics:
    """Modeled step walltime (workload.py:314-363).  run_simulation computes
    the same columns natively; this host version serves library users."""
    model = resolve_costs(cfg)
    a, b = faces if faces is not None else ba.interior_faces()
    split = dm.owner[a] != dm.owner[b]
    nf = (np.bincount(dm.owner[a][split], minlength=dm.n_ranks)
          + np.bincount(dm.owner[b][split], minlength=dm.n_ranks))
    compute_max = float(np.max(rank_compute)) * overhead
    comm_max = float(nf.max()) * model.comm_per_face * overhead
    gather = (model.gather if outcome.attempted else 0.0) * overhead
    redis = 0.0
    if outcome.adopted:
        moved = int(state.per_box_particles[dm.owner != prev_dm.owner].sum())
        redis = model.redistribute_latency + model.redistribute_per_particle * moved
    redis *= overhead
    occ = np.bincount(dm.owner, weights=state.per_box_particles, minlength=dm.n_ranks)
    mrp = int(occ.max())
    return StepMetrics(
        step=state.step - 1, efficiency_before=outcome.efficiency_current,
        efficiency_after=(outcome.efficiency_proposed if outcome.adopted
                          else outcome.efficiency_current),
        adopted=outcome.adopted, compute_max=compute_max, comm_max=comm_max,
        gather=gather, redistribute=redis,
        walltime=compute_max + comm_max + gather + redis, max_rank_particles=mrp,
        oom=cfg.capacity_particles is not None and mrp > cfg.capacity_particles)


def initial_mapping(cfg: ScenarioConfig, ba: BoxArray, state_or_counts) -> DistributionMapping:
    from .balancer import knapsack_assign, sfc_assign

    if cfg.initial_mapping == "slab":
        return slab_mapping(ba, cfg.n_ranks)
    if cfg.initial_mapping == "roundrobin":
        return round_robin_mapping(ba, cfg.n_ranks)
    work = CostVector(values=true_work(state_or_counts, cfg), step=0)
    if cfg.initial_mapping == "knapsack":
        return knapsack_assign(work, cfg.n_ranks)
    return sfc_assign(work, morton_order(ba), cfg.n_ranks)


def policy_kind(policy: BalancePolicy, total_steps: int) -> str:
    if policy.interval <= total_steps:
        return "dynamic"
    return "static" if policy.static_step is not None else "none"


PIC_DEFAULTS = {"dt": 0.5, "q_over_m": -1.0, "q_times_w": -1e-4}


def sim_config(cfg: ScenarioConfig, policy: BalancePolicy, provider: CostProvider,
               physics: str = "surrogate", pic: dict | None = None):
    """Flatten (scenario, policy, provider) into lbx_sim_config."""
    if provider.device_kind < 0 or provider.device_kind > 5:
        raise ConfigError(f"provider {provider.kind!r} is not supported by the native loop")
    model = resolve_costs(cfg)
    w = getattr(provider, "weights", None)
    mc = getattr(provider, "cfg", None)
    return _lib.SimConfig(
        extent_z=cfg.domain_extent[0], extent_x=cfg.domain_extent[1],
        box_size=cfg.box_size, n_ranks=cfg.n_ranks, total_steps=cfg.total_steps,
        kick_step=cfg.kick.step,
        strategy=0 if policy.strategy is Strategy.KNAPSACK else 1,
        interval=policy.interval, improvement_threshold=policy.improvement_threshold,
        threshold_relative=1 if policy.threshold_mode == "relative" else 0,
        cap_factor=policy.knapsack_cap_factor,
        static_step=-1 if policy.static_step is None else policy.static_step,
        cost_kind=provider.device_kind,
        w_particle=w.w_particle if w else 0.75, w_cell=w.w_cell if w else 0.25,
        noise_amplitude=mc.noise_amplitude if mc else 0.0,
        noise_seed=mc.seed if mc else 0, overhead_factor=provider.overhead_factor,
        work_wp=cfg.work_weights[0], work_wc=cfg.work_weights[1],
        comm_per_face=model.comm_per_face, gather=model.gather,
        redistribute_per_particle=model.redistribute_per_particle,
        redistribute_latency=model.redistribute_latency,
        capacity_particles=-1 if cfg.capacity_particles is None else cfg.capacity_particles,
        physics=0 if physics == "surrogate" else 1,
        pic_dt=(pic or PIC_DEFAULTS)["dt"], pic_q_over_m=(pic or PIC_DEFAULTS)["q_over_m"],
        pic_q_times_w=(pic or PIC_DEFAULTS)["q_times_w"], extent_y=0,
        migration_ratio=getattr(policy, "migration_ratio", 0.0),
        clock_mode=getattr(provider, "clock_mode", 0))


class Simulation:
    """Device-resident run: particles in HBM (SoA), native stepping loop.

    ``Simulation(cfg, policy, provider).run()`` == run_simulation(...);
    ``run(first, last)`` runs a sub-range (benchmarks time a window).
    ``physics="pic"`` replaces the reference's ballistic advance with the
    2D3V PIC step (pic.py); the kick then sets momenta u = v_kick / dt."""

    def __init__(self, cfg: ScenarioConfig, policy: BalancePolicy, provider: CostProvider,
                 *, device="cuda:0", positions=None, kick=None, initial_owner=None,
                 record_counts=False, record_clock=False, time_kernels=False,
                 physics="surrogate", pic=None):
        import torch

        from . import device as D

        self.cfg, self.policy, self.provider = cfg, policy, provider
        self.dev = D.require_cuda(device)
        self.ba = box_array_for(cfg)
        pos = sample_blob(cfg) if positions is None else positions
        self.n_init = n = int(pos.shape[0])
        self.ctx = D.Context(self.dev, capacity=n)
        self.state = D.ParticleState.empty(n, self.dev)
        if isinstance(pos, torch.Tensor):
            self.state.z[:n].copy_(pos[:, 0])
            self.state.x[:n].copy_(pos[:, 1])
        else:
            self.state.load(pos, np.zeros_like(pos))
        self.state.n = n
        nbz, nbx = self.ba.grid_shape
        counts0 = D.bin_aos(torch.stack([self.state.z[:n], self.state.x[:n]], 1).contiguous(),
                            cfg.box_size, nbz, nbx).cpu().numpy()
        self.counts0 = counts0
        if initial_owner is None:
            initial_owner = initial_mapping(cfg, self.ba, counts0).owner
        self.initial_owner = np.array(initial_owner, dtype=np.int64)
        self.kvz = self.kvx = None
        if cfg.kick.step < cfg.total_steps:
            if kick is None:
                kick = kick_velocities(pos if isinstance(pos, np.ndarray)
                                       else pos.cpu().numpy(), cfg)
            kick = kick if isinstance(kick, torch.Tensor) else torch.from_numpy(kick)
            self.kvz = torch.zeros(n + 2, dtype=torch.float64, device=self.dev)
            self.kvx = torch.zeros(n + 2, dtype=torch.float64, device=self.dev)
            self.kvz[:n].copy_(kick[:, 0])
            self.kvx[:n].copy_(kick[:, 1])
        self.physics = physics
        self.pic = dict(PIC_DEFAULTS, **(pic or {}))
        if physics == "pic" and self.kvz is not None:   # momenta from the kick
            self.kvz.div_(self.pic["dt"])
            self.kvx.div_(self.pic["dt"])
        self.conf = sim_config(cfg, policy, provider, physics, self.pic)
        h = C.c_void_p()
        _lib.check(_lib.lib.lbx_sim_create(C.byref(h), self.ctx.handle, C.byref(self.conf)))
        self.handle = h
        st = self.state
        _lib.check(_lib.lib.lbx_sim_set_particles(
            h, _lib.ptr(st.z), _lib.ptr(st.x), _lib.ptr(st.vz), _lib.ptr(st.vx),
            _lib.ptr(self.kvz), _lib.ptr(self.kvx), n, D._stream(self.dev)))
        if physics == "pic":
            from .pic import CURRENT_NAMES, FIELD_NAMES
            nz, nx = cfg.domain_extent
            self.fields = {k: torch.zeros((nz + 2, nx + 2), dtype=torch.float32,
                                          device=self.dev) for k in FIELD_NAMES + CURRENT_NAMES}
            self.uy = torch.zeros(n + 2, dtype=torch.float64, device=self.dev)
            fa = (C.c_void_p * 6)(*(_lib.ptr(self.fields[k]) for k in FIELD_NAMES))
            ca = (C.c_void_p * 3)(*(_lib.ptr(self.fields[k]) for k in CURRENT_NAMES))
            _lib.check(_lib.lib.lbx_sim_set_fields(h, fa, ca, _lib.ptr(self.uy)))
        T, nb = cfg.total_steps, self.ba.n_boxes
        self.out = {k: np.zeros(T) for k in ("eff_before", "eff_after", "compute_max",
                                             "comm_max", "gather", "redistribute",
                                             "walltime", "kernel_ms")}
        for k in ("adopted", "attempted", "oom"):
            self.out[k] = np.zeros(T, dtype=np.uint8)
        self.out["max_rank_particles"] = np.zeros(T, dtype=np.int64)
        self.out["n_alive"] = np.zeros(T, dtype=np.int64)
        self.out["cost_trace"] = np.zeros((T, nb))
        self.out["count_trace"] = np.zeros((T, nb), dtype=np.int64) if record_counts else None
        self.out["clock_trace"] = np.zeros((T, nb), dtype=np.uint64) if record_clock else None
        self.out["owner"] = self.initial_owner.copy()
        self.out["adopt_steps"] = np.zeros(T, dtype=np.int64)
        self.out["adopt_owners"] = np.zeros((T, nb), dtype=np.int64)
        for v in self.out.values():   # fault the pages in now, not inside the native loop
            if v is not None:
                v.fill(0)
        self.out["owner"][:] = self.initial_owner
        self.time_kernels = time_kernels
        o = self.out
        self.souts = _lib.SimOutputs(
            *(_lib.ptr(o[k]) for k in ("eff_before", "eff_after", "adopted", "attempted",
                                       "compute_max", "comm_max", "gather", "redistribute",
                                       "walltime", "max_rank_particles", "oom", "n_alive",
                                       "cost_trace", "count_trace", "clock_trace", "owner",
                                       "adopt_steps", "adopt_owners")),
            _lib.ptr(o["kernel_ms"]) if time_kernels else None, 0, 0, 0)
        self.done = 0

    def run(self, first: int | None = None, last: int | None = None):
        from .device import _stream

        first = self.done if first is None else first
        last = self.cfg.total_steps if last is None else last
        _lib.check(_lib.lib.lbx_sim_run(self.handle, first, last, C.byref(self.souts),
                                        _stream(self.dev)))
        self.done = max(self.done, int(self.souts.completed_steps))
        return self

    @property
    def graph_cycles(self) -> int:
        """16-step cycles the native loop has replayed as CUDA graphs."""
        out = C.c_int64()
        _lib.check(_lib.lib.lbx_sim_graph_cycles(self.handle, C.byref(out)))
        return out.value

    @property
    def resident_runs(self) -> int:
        """run() calls the native loop executed on the resident kernel."""
        out = C.c_int64()
        _lib.check(_lib.lib.lbx_sim_resident_runs(self.handle, C.byref(out)))
        return out.value

    def close(self):
        if getattr(self, "handle", None):
            _lib.lib.lbx_sim_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def live_particles(self) -> int:
        return self.ctx.count()

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
        snaps = [(int(o["adopt_steps"][i]), o["adopt_owners"][i].copy()) for i in range(na)]
        eff = np.array([m.efficiency_after for m in metrics])
        oom = bool(done and metrics[-1].oom)
        final = int(o["n_alive"][done - 1]) if done else self.n_init
        from .device import ParticleState
        kicked = self.kvz is not None and done > cfg.kick.step
        st = self.state
        final_state = ParticleState(st.z, st.x, self.kvz if kicked else st.vz,
                                    self.kvx if kicked else st.vx, final)
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
            "oom": oom, "final_particles": final,
        }
        return RunResult(
            metrics=metrics, summary=summary, cost_trace=o["cost_trace"][:done].copy(),
            initial_owner=self.initial_owner.copy(), adoption_snapshots=snaps,
            n_alive=o["n_alive"][:done].copy(),
            count_trace=None if o["count_trace"] is None else o["count_trace"][:done].copy(),
            clock_trace=None if o["clock_trace"] is None else o["clock_trace"][:done].copy(),
            kernel_ms=o["kernel_ms"][:done].copy() if self.time_kernels else None,
            final_state=final_state)


def run_simulation(cfg: ScenarioConfig, policy: BalancePolicy, provider: CostProvider,
                   **kw) -> RunResult:
    """Advance, assess, balance and price every step (workload.py:388-470);
    halts with OOM status when a rank's particles exceed capacity."""
    sim = Simulation(cfg, policy, provider, **kw)
    try:
        sim.run()
        return sim.result()
    finally:
        sim.close()
