"""Load-balance efficiency, mapping policies and the gated adoption rule --
API mirror of lbsim/balancer.py backed by libLBX's C++ balancer.

Efficiency E = mean(rank load) / max(rank load).  Knapsack = greedy LPT
under a per-rank box cap followed by 1-for-1 swap refinement; SFC = greedy
contiguous split of the Morton curve.  A proposal is adopted only if it
improves E by the threshold (relative by default) and never if it is worse.
All arithmetic is bit-exact with the reference (see lbx_balancer.cpp).
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cost import CostVector
from .decomposition import DistributionMapping
from .errors import ConfigError


class Strategy(enum.Enum):
    KNAPSACK = "knapsack"
    SFC = "sfc"


@dataclass(frozen=True)
class BalancePolicy:
    """When to attempt a rebalance and with which policy (balancer.py:31-59).

    Attempts run at steps 0, interval, 2*interval, ...; interval > run
    length disables them (no load balancing); static_step forces one
    attempt (static load balancing)."""

    strategy: Strategy = Strategy.KNAPSACK
    interval: int = 10
    improvement_threshold: float = 0.10
    knapsack_cap_factor: float = 1.5
    threshold_mode: str = "relative"
    static_step: int | None = None
    # B200 extension: >0 also requires the load saved over
    # one interval to exceed the migration cost (migration_ratio particle-
    # pushes per moved particle).  0 = the reference's gate.
    migration_ratio: float = 0.0
    # B200 extension: the distributed loop MEASURES every adoption's
    # redistribution (wall time of partition -> exchange -> unpack, max over
    # ranks) and the step's push time, and sets migration_ratio to their
    # per-particle ratio (pushes per moved particle) for later adoptions.
    measured_migration: bool = False

    def __post_init__(self):
        if self.migration_ratio < 0:
            raise ConfigError("migration_ratio must be >= 0")
        if self.interval < 1:
            raise ConfigError(f"interval must be >= 1, got {self.interval}")
        if self.improvement_threshold < 0:
            raise ConfigError("improvement_threshold must be >= 0")
        if self.knapsack_cap_factor < 1:
            raise ConfigError("knapsack_cap_factor must be >= 1")
        if self.threshold_mode not in ("relative", "absolute"):
            raise ConfigError("threshold_mode must be 'relative' or 'absolute', "
                              f"got {self.threshold_mode!r}")


@dataclass(frozen=True)
class BalanceOutcome:
    proposed: DistributionMapping
    efficiency_current: float
    efficiency_proposed: float
    adopted: bool
    attempted: bool = True


def _vec(costs: CostVector, dm: DistributionMapping):
    if costs.n_boxes != dm.n_boxes:
        raise ValueError(f"cost vector length {costs.n_boxes} does not match mapping "
                         f"length {dm.n_boxes}")
    return np.ascontiguousarray(costs.values), np.ascontiguousarray(dm.owner)


def rank_loads(costs: CostVector, dm: DistributionMapping) -> np.ndarray:
    v, own = _vec(costs, dm)
    out = np.zeros(dm.n_ranks)
    _lib.check(_lib.lib.lbx_rank_loads(_lib.ptr(v), _lib.ptr(own), v.size, dm.n_ranks,
                                       _lib.ptr(out)))
    return out


def efficiency_flagged(costs: CostVector, dm: DistributionMapping) -> tuple[float, bool]:
    """(E, degenerate): all-zero loads report (1.0, True)."""
    v, own = _vec(costs, dm)
    e, d = C.c_double(), C.c_int32()
    _lib.check(_lib.lib.lbx_efficiency(_lib.ptr(v), _lib.ptr(own), v.size, dm.n_ranks,
                                       C.byref(e), C.byref(d)))
    return float(e.value), bool(d.value)


def efficiency(costs: CostVector, dm: DistributionMapping) -> float:
    return efficiency_flagged(costs, dm)[0]


def knapsack_assign(costs: CostVector, n_ranks: int,
                    cap_factor: float = 1.5) -> DistributionMapping:
    """Locality-blind greedy + swap refinement, cap ceil(cap*boxes/ranks)."""
    v = np.ascontiguousarray(costs.values)
    out = np.empty(v.size, dtype=np.int64)
    _lib.check(_lib.lib.lbx_knapsack(_lib.ptr(v), v.size, int(n_ranks), float(cap_factor),
                                     _lib.ptr(out)))
    return DistributionMapping(owner=out, n_ranks=n_ranks)


def sfc_assign(costs: CostVector, curve, n_ranks: int) -> DistributionMapping:
    """Contiguous segments of the curve, greedy against total/n_ranks."""
    v = np.ascontiguousarray(costs.values)
    cv = np.ascontiguousarray(curve, dtype=np.int64)
    if cv.size != v.size and v.size:
        raise ValueError("curve must be a permutation of box indices")
    out = np.empty(v.size, dtype=np.int64)
    _lib.check(_lib.lib.lbx_sfc(_lib.ptr(v), _lib.ptr(cv), v.size, int(n_ranks),
                                _lib.ptr(out)))
    return DistributionMapping(owner=out, n_ranks=n_ranks)


def sfc_assign_optimal(costs: CostVector, curve, n_ranks: int) -> DistributionMapping:
    """Exact min-max contiguous split of the curve (balancer.py:222-255):
    a validation reference for the greedy split, not on the stepping path."""
    cv = np.asarray(curve, dtype=np.int64)
    n = cv.size
    if n == 0:
        raise ValueError("cannot partition an empty cost vector")
    k_eff = min(n_ranks, n)
    pre = np.concatenate(([0.0], np.cumsum(costs.values[cv])))
    best = pre[1:].copy()
    cut = np.zeros((k_eff, n + 1), dtype=np.int64)
    for k in range(1, k_eff):
        nxt = np.full(n, np.inf)
        for i in range(k + 1, n + 1):
            j = np.arange(k, i)
            c = np.maximum(best[j - 1], pre[i] - pre[j])
            m = int(np.argmin(c))
            nxt[i - 1] = c[m]
            cut[k, i] = j[m]
        best = nxt
    owner = np.empty(n, dtype=np.int64)
    end = n
    for k in range(k_eff - 1, -1, -1):
        start = int(cut[k, end]) if k else 0
        owner[cv[start:end]] = k
        end = start
    return DistributionMapping(owner=owner, n_ranks=n_ranks)


def gate(e_cur: float, e_prop: float, policy: BalancePolicy) -> bool:
    """Adoption rule of balancer.py:285-289."""
    if policy.threshold_mode == "relative":
        need = e_cur * (1.0 + policy.improvement_threshold)
    else:
        need = e_cur + policy.improvement_threshold
    return bool(e_prop >= need and e_prop >= e_cur)


def migration_worthwhile(costs: CostVector, current: DistributionMapping,
                         proposed: DistributionMapping, counts, policy: BalancePolicy) -> bool:
    """The migration-aware part of the gate (B200 extension, SURVEY 8f rank
    3), the same arithmetic as lbx_runtime.cpp's lb_step: the max-rank load
    saved over one interval must exceed migration_ratio x (cost per particle)
    x (particles in boxes that change owner)."""
    c = np.asarray(costs.values, dtype=np.float64)
    n = np.asarray(counts, dtype=np.int64)
    if n.shape != c.shape:
        raise ValueError(f"counts length {n.size} != costs length {c.size}")
    R = current.n_ranks
    lc, lp = [0.0] * R, [0.0] * R
    total_cost, total_n, moved = 0.0, 0, 0
    for b in range(c.size):            # box order, as the C++ loop
        lc[int(current.owner[b])] += float(c[b])
        lp[int(proposed.owner[b])] += float(c[b])
        total_cost += float(c[b])
        total_n += int(n[b])
        if proposed.owner[b] != current.owner[b]:
            moved += int(n[b])
    per_push = total_cost / float(total_n) if total_n > 0 else 0.0
    saved = float(policy.interval) * (max(lc) - max(lp))
    return saved > policy.migration_ratio * per_push * float(moved)


def attempt_rebalance(costs: CostVector, current: DistributionMapping,
                      policy: BalancePolicy, step: int, *, curve=None,
                      force: bool = False, counts=None) -> BalanceOutcome:
    """One pass of the balancing routine (balancer.py:258-292).  With
    policy.migration_ratio > 0 the per-box particle `counts` are required
    and the migration-aware check (migration_worthwhile) joins the gate,
    exactly as in the native loop."""
    if step < 0:
        raise ValueError(f"step must be >= 0, got {step}")
    if policy.migration_ratio > 0 and counts is None:
        raise ValueError("migration_ratio > 0 needs the per-box particle counts")
    e_cur = efficiency(costs, current)
    if not force and step % policy.interval:
        return BalanceOutcome(current, e_cur, e_cur, adopted=False, attempted=False)
    if policy.strategy is Strategy.KNAPSACK:
        prop = knapsack_assign(costs, current.n_ranks, policy.knapsack_cap_factor)
    else:
        if curve is None:
            raise ValueError("sfc strategy requires the morton curve")
        prop = sfc_assign(costs, curve, current.n_ranks)
    e_prop = efficiency(costs, prop)
    adopted = gate(e_cur, e_prop, policy)
    if adopted and policy.migration_ratio > 0:
        adopted = migration_worthwhile(costs, current, prop, counts, policy)
    return BalanceOutcome(prop, e_cur, e_prop, adopted=adopted)


def periodic_enabled(policy: BalancePolicy, total_steps: int) -> bool:
    return policy.interval <= total_steps


def should_attempt(policy: BalancePolicy, step: int, total_steps: int) -> bool:
    """Attempt schedule (balancer.py:300-304)."""
    if policy.static_step is not None and step == policy.static_step:
        return True
    return periodic_enabled(policy, total_steps) and step % policy.interval == 0
