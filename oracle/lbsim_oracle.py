"""CPU oracle for the lbsim hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference simulator's per-step
path (arXiv 2104.11385 reference package ``lbsim`` under
``/root/reference/pkg/src/lbsim``).  It exists so that the CUDA/C++ product
path can be checked on a machine where the reference itself is absent (the
GPU box).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu-baseline / reference arm may import it, and only as the checker or the
timed CPU baseline -- never as the product.

Pinning: every function here is checked against the reference run in-process
(``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src`` and
writes fixtures; ``tests/test_oracle.py`` compares this module against those
fixtures and against the known answers in the reference's own tests).

Each function cites the reference file:line whose arithmetic it restates.
Floating-point expression order is kept exactly (no re-association), since
the product must be bit-exact with it.
"""

from __future__ import annotations

import math

import numpy as np

# workload.py:34-37
SKIRT_CUTOFF = 12.0
SEED_INIT = 1
SEED_KICK = 2
# cost.py:111 (stream key of the simulated on-device timer)
MEASURE_KEY = 0x6D656173
# cost.py:21-24
WEIGHTS = {"default": (0.75, 0.25), "sfc": (0.02, 0.98)}


# ----------------------------------------------------------------------------
# L0 kernels
# ----------------------------------------------------------------------------

def advance_particles(pos, vel, ez, ex):
    """_kernels.pyx:12-35 / _kernels_py.py:13-22.

    new = pos + vel; a particle survives iff 0 <= new < extent on both axes;
    survivors keep their order and their (old) velocities.
    """
    pos = np.asarray(pos, dtype=np.float64).reshape(-1, 2)
    vel = np.asarray(vel, dtype=np.float64).reshape(-1, 2)
    nz = pos[:, 0] + vel[:, 0]
    nx = pos[:, 1] + vel[:, 1]
    alive = (nz >= 0.0) & (nz < ez) & (nx >= 0.0) & (nx < ex)
    out_pos = np.stack([nz[alive], nx[alive]], axis=1)
    return np.ascontiguousarray(out_pos), np.ascontiguousarray(vel[alive])


def bin_particles(pos, box_size, nbz, nbx):
    """_kernels.pyx:38-47: count[(int)(z/M)*nbx + (int)(x/M)] += 1.

    IEEE division then truncation toward zero (== floor, positions >= 0).
    """
    pos = np.asarray(pos, dtype=np.float64).reshape(-1, 2)
    bz = np.trunc(pos[:, 0] / box_size).astype(np.int64)
    bx = np.trunc(pos[:, 1] / box_size).astype(np.int64)
    ids = bz * nbx + bx
    return np.bincount(ids, minlength=nbz * nbx).astype(np.int64)


# ----------------------------------------------------------------------------
# L2 cost assessment
# ----------------------------------------------------------------------------

def heuristic_cost(counts, cells, wp, wc):
    """cost.py:83-95: wp*particles + wc*cells, two products then one add."""
    p = np.asarray(counts, dtype=np.float64)
    c = np.asarray(cells, dtype=np.float64)
    return wp * p + wc * c


def true_work(counts, box_size, w):
    """workload.py:303-311."""
    cells = float(box_size * box_size)
    return w[0] * np.asarray(counts).astype(np.float64) + w[1] * cells


def measured_cost(work, amplitude, seed, step):
    """cost.py:98-113: work * (1 + U[-a, a]) from PCG64 keyed (seed, 'meas', step)."""
    work = np.asarray(work, dtype=np.float64)
    if amplitude == 0.0:
        return work.copy()
    gen = np.random.default_rng((int(seed), MEASURE_KEY, int(step)))
    eps = gen.uniform(-amplitude, amplitude, size=work.size)
    return work * (1.0 + eps)


# ----------------------------------------------------------------------------
# L1 decomposition
# ----------------------------------------------------------------------------

def morton_code(a, b):
    """decomposition.py:137-159: bits of a on even positions, b on odd."""
    code = 0
    bit = 0
    while a or b:
        code |= (a & 1) << (2 * bit)
        code |= (b & 1) << (2 * bit + 1)
        a >>= 1
        b >>= 1
        bit += 1
    return code


def morton_order(nbz, nbx):
    """decomposition.py:162-168: stable argsort of the box codes."""
    codes = np.array([morton_code(i // nbx, i % nbx) for i in range(nbz * nbx)],
                     dtype=np.int64)
    return np.argsort(codes, kind="stable").astype(np.int64)


def slab_mapping(n_boxes, n_ranks):
    """decomposition.py:176-181."""
    edges = np.linspace(0, n_boxes, n_ranks + 1)
    owner = np.searchsorted(edges, np.arange(n_boxes), side="right") - 1
    return np.clip(owner, 0, n_ranks - 1).astype(np.int64)


def round_robin_mapping(n_boxes, n_ranks):
    """decomposition.py:184-187."""
    return np.arange(n_boxes, dtype=np.int64) % n_ranks


def interior_faces(nbz, nbx):
    """decomposition.py:71-81: vertical neighbours first, then horizontal."""
    grid = np.arange(nbz * nbx, dtype=np.int64).reshape(nbz, nbx)
    lo = np.concatenate([grid[:-1, :].ravel(), grid[:, :-1].ravel()])
    hi = np.concatenate([grid[1:, :].ravel(), grid[:, 1:].ravel()])
    return lo, hi


# ----------------------------------------------------------------------------
# L3 balancer
# ----------------------------------------------------------------------------

def rank_loads(cost, owner, n_ranks):
    """balancer.py:73-79: bincount with weights (sequential, box order)."""
    return np.bincount(np.asarray(owner, dtype=np.int64),
                       weights=np.asarray(cost, dtype=np.float64),
                       minlength=n_ranks)


def efficiency_flagged(cost, owner, n_ranks):
    """balancer.py:82-93: pairwise mean over max; all-zero -> (1.0, True)."""
    loads = rank_loads(cost, owner, n_ranks)
    top = loads.max()
    if top == 0.0:
        return 1.0, True
    return float(loads.mean() / top), False


def knapsack_assign(cost, n_ranks, cap_factor=1.5):
    """balancer.py:102-134 (+ _refine_by_swaps 137-179)."""
    if n_ranks < 1:
        raise ValueError(f"n_ranks must be >= 1, got {n_ranks}")
    v = np.asarray(cost, dtype=np.float64)
    n = v.size
    cap = math.ceil(cap_factor * n / n_ranks) if n else 0
    if cap * n_ranks < n:
        raise ValueError(f"box cap {cap} per rank too tight")
    order = np.lexsort((np.arange(n), -v))
    owner = np.empty(n, dtype=np.int64)
    loads = np.zeros(n_ranks)
    nbox = np.zeros(n_ranks, dtype=np.int64)
    for b in order:
        r = int(np.argmin(np.where(nbox < cap, loads, np.inf)))
        owner[b] = r
        loads[r] += v[b]
        nbox[r] += 1
    _swap_refine(owner, loads, v, n_ranks)
    return owner


def _swap_refine(owner, loads, v, n_ranks):
    """balancer.py:137-179: best 1-for-1 swap off the unique max rank."""
    if n_ranks < 2 or v.size < 2:
        return
    while True:
        top = loads.max()
        at_top = np.flatnonzero(loads == top)
        if at_top.size != 1:
            return
        rmax = int(at_top[0])
        mine = np.flatnonzero(owner == rmax)
        rest = np.flatnonzero(owner != rmax)
        if mine.size == 0 or rest.size == 0:
            return
        rest_load = loads[owner[rest]]
        rest_v = v[rest]
        found = None
        for a in mine:
            va = v[a]
            here = top - va + rest_v
            there = rest_load - rest_v + va
            worst = np.maximum(here, there)
            ok = np.flatnonzero(worst < top)
            if ok.size == 0:
                continue
            j = ok[np.argmin(worst[ok])]
            if found is None or worst[j] < found[0]:
                found = (worst[j], int(a), int(rest[j]))
        if found is None:
            return
        _, a, b = found
        rb = int(owner[b])
        loads[rmax] += v[b] - v[a]
        loads[rb] += v[a] - v[b]
        owner[a] = rb
        owner[b] = rmax


def sfc_assign(cost, curve, n_ranks):
    """balancer.py:182-219: greedy contiguous split of the Morton curve."""
    if n_ranks < 1:
        raise ValueError(f"n_ranks must be >= 1, got {n_ranks}")
    curve = np.asarray(curve, dtype=np.int64)
    n = curve.size
    if n == 0:
        raise ValueError("cannot partition an empty cost vector")
    if not np.array_equal(np.sort(curve), np.arange(n)):
        raise ValueError("curve must be a permutation of box indices")
    seq = np.asarray(cost, dtype=np.float64)[curve]
    target = seq.sum() / n_ranks
    owner = np.empty(n, dtype=np.int64)
    pos = 0
    for r in range(n_ranks):
        if pos == n:
            break
        if r == n_ranks - 1:
            owner[curve[pos:]] = r
            break
        first = pos
        acc = seq[pos]
        pos += 1
        keep_back = n_ranks - r - 1
        while pos < n - keep_back:
            nxt = seq[pos]
            if abs(acc + nxt - target) > abs(acc - target):
                break
            acc += nxt
            pos += 1
        owner[curve[first:pos]] = r
    return owner


def sfc_assign_optimal(cost, curve, n_ranks):
    """balancer.py:222-255: exact min-max contiguous split (DP)."""
    curve = np.asarray(curve, dtype=np.int64)
    n = curve.size
    if n == 0:
        raise ValueError("cannot partition an empty cost vector")
    k_max = min(n_ranks, n)
    pre = np.concatenate(([0.0], np.cumsum(np.asarray(cost, float)[curve])))
    best = pre[1:].copy()
    cut = np.zeros((k_max, n + 1), dtype=np.int64)
    for k in range(1, k_max):
        nxt = np.empty(n)
        for i in range(k + 1, n + 1):
            j = np.arange(k, i)
            c = np.maximum(best[j - 1], pre[i] - pre[j])
            m = int(np.argmin(c))
            nxt[i - 1] = c[m]
            cut[k][i] = j[m]
        nxt[:k] = np.inf
        best = nxt
    owner = np.empty(n, dtype=np.int64)
    end = n
    for k in range(k_max - 1, -1, -1):
        start = cut[k][end] if k else 0
        owner[curve[start:end]] = k
        end = start
    return owner


def gate(e_cur, e_prop, threshold, mode):
    """balancer.py:285-289."""
    need = e_cur * (1.0 + threshold) if mode == "relative" else e_cur + threshold
    return bool(e_prop >= need and e_prop >= e_cur)


def should_attempt(interval, static_step, step, total_steps):
    """balancer.py:295-304."""
    if static_step is not None and step == static_step:
        return True
    return interval <= total_steps and step % interval == 0


# ----------------------------------------------------------------------------
# L4 workload
# ----------------------------------------------------------------------------

def init_scenario(extent, box_size, center, core, edge, ppc, seed):
    """workload.py:218-269; returns (positions [n,2], per-box counts)."""
    nz, nx = extent
    reach = core + SKIRT_CUTOFF * edge + 1.0
    iz, ix = np.meshgrid(np.arange(nz), np.arange(nx), indexing="ij")
    iz = iz.ravel()
    ix = ix.ravel()
    near = np.hypot(iz + 0.5 - center[0], ix + 0.5 - center[1]) <= reach
    iz, ix = iz[near], ix[near]
    if iz.size == 0 or ppc == 0:
        raise ValueError("scenario produces zero particles")
    gen = np.random.default_rng((int(seed), SEED_INIT))
    whole = int(math.floor(ppc))
    part = ppc - whole
    per_cell = np.full(iz.size, whole, dtype=np.int64)
    if part > 0.0:
        per_cell += gen.random(iz.size) < part
    total = int(per_cell.sum())
    if total == 0:
        raise ValueError("scenario produces zero particles")
    oz = np.repeat(iz, per_cell).astype(np.float64)
    ox = np.repeat(ix, per_cell).astype(np.float64)
    u = gen.random((total, 2))
    pos = np.column_stack((oz + u[:, 0], ox + u[:, 1]))
    rho = np.hypot(pos[:, 0] - center[0], pos[:, 1] - center[1])
    if edge > 0.0:
        p_keep = np.where(rho <= core, 1.0, np.exp(-(rho - core) / edge))
    else:
        p_keep = (rho <= core).astype(np.float64)
    pos = np.ascontiguousarray(pos[gen.random(total) < p_keep])
    if pos.shape[0] == 0:
        raise ValueError("scenario produces zero particles")
    counts = bin_particles(pos, float(box_size), nz // box_size, nx // box_size)
    return pos, counts


def kick_velocities(pos, center, speed, drift, seed):
    """workload.py:272-283."""
    gen = np.random.default_rng((int(seed), SEED_KICK))
    f = gen.uniform(0.5, 1.5, size=pos.shape[0])
    dz = pos[:, 0] - center[0]
    dx = pos[:, 1] - center[1]
    rho = np.hypot(dz, dx)
    uz = np.divide(dz, rho, out=np.zeros_like(dz), where=rho > 0)
    ux = np.divide(dx, rho, out=np.zeros_like(dx), where=rho > 0)
    s = speed * f
    return np.ascontiguousarray(np.column_stack((s * uz + drift, s * ux)))


def resolve_costs(cfg):
    """workload.py:180-215: derived walltime-model coefficients."""
    if cfg.get("costs") is not None:
        c = cfg["costs"]
        return (c["comm_per_face"], c["gather"], c["redistribute_per_particle"],
                c["redistribute_latency"])
    nz, nx = cfg["extent"]
    r, s = cfg["core_radius"], cfg["edge_scale"]
    est_p = cfg["ppc"] * (math.pi * r * r + 2.0 * math.pi * r * s)
    wp, wc = cfg["work_weights"]
    c_avg = (wp * est_p + wc * (nz * nx)) / cfg["ranks"]
    w_est = c_avg / cfg["compute_fraction"]
    nbz, nbx = nz // cfg["box_size"], nx // cfg["box_size"]
    faces = 2 * nbz * nbx - nbz - nbx
    per_rank = max(2.0 * faces / cfg["ranks"] * (1.0 - 1.0 / cfg["ranks"]), 1.0)
    comm = c_avg * (1.0 - cfg["compute_fraction"]) / cfg["compute_fraction"]
    return (comm / per_rank, 0.025 * w_est, 3.0 * w_est / max(est_p, 1.0),
            0.05 * w_est)


def config_from_doc(doc):
    """Flatten a scenario YAML document (scenarios.py:58-133 schema)."""
    dom = doc["domain"]
    blob = doc["blob"]
    kick = doc["kick"]
    bal = doc.get("balance", {}) or {}
    prov = doc.get("provider", {}) or {}
    w = prov.get("weights", "default")
    if isinstance(w, str):
        w = WEIGHTS[w]
    return dict(
        scenario_id=str(doc["scenario_id"]),
        extent=(int(dom["extent"][0]), int(dom["extent"][1])),
        box_size=int(dom["box_size"]), ranks=int(doc["ranks"]),
        center=(float(blob["center"][0]), float(blob["center"][1])),
        core_radius=float(blob["core_radius"]),
        edge_scale=float(blob.get("edge_scale", 0.0)),
        ppc=float(blob["particles_per_cell"]),
        kick_step=int(kick["step"]), kick_speed=float(kick["speed"]),
        kick_drift=float(kick.get("drift", 0.0)),
        steps=int(doc["steps"]),
        compute_fraction=float(doc.get("compute_fraction", 0.5)),
        work_weights=tuple(float(v) for v in doc.get("work_weights", [0.75, 0.25])),
        costs=doc.get("costs"),
        capacity=doc.get("capacity_particles"),
        initial_mapping=str(doc.get("initial_mapping", "slab")),
        seed=int(doc.get("seed", 1)),
        strategy=str(bal.get("strategy", "knapsack")),
        interval=int(bal.get("interval", 10)),
        threshold=float(bal.get("threshold", 0.10)),
        cap_factor=float(bal.get("cap_factor", 1.5)),
        threshold_mode=str(bal.get("threshold_mode", "relative")),
        static_step=bal.get("static_step"),
        provider=str(prov.get("kind", "heuristic")),
        provider_weights=tuple(float(v) for v in w),
        noise=float(prov.get("noise", 0.05)),
        instrumented_overhead=float(prov.get("instrumented_overhead", 2.0)),
    )


def apply_policy(cfg, policy):
    """scenarios.py:163-177 (--policy none|static|knapsack|sfc)."""
    cfg = dict(cfg)
    off = cfg["steps"] + 1
    if policy == "none":
        cfg.update(interval=off, static_step=None)
    elif policy == "static":
        cfg.update(interval=off,
                   static_step=0 if cfg["static_step"] is None else cfg["static_step"])
    elif policy in ("knapsack", "sfc"):
        cfg.update(strategy=policy, static_step=None)
        if cfg["interval"] > cfg["steps"]:
            cfg["interval"] = 10
    else:
        raise ValueError(policy)
    return cfg


def run_simulation(cfg, *, record_counts=False, record_positions_at=()):
    """workload.py:388-470: the whole stepping loop, returning plain arrays.

    Returns a dict with per-step metric columns, the cost trace, the initial
    owner vector, adoption snapshots and the summary scalars.
    """
    nz, nx = cfg["extent"]
    m = cfg["box_size"]
    nbz, nbx = nz // m, nx // m
    nb = nbz * nbx
    R = cfg["ranks"]
    curve = morton_order(nbz, nbx)
    fa, fb = interior_faces(nbz, nbx)
    cells = np.full(nb, m * m, dtype=np.int64)
    pos, counts = init_scenario(cfg["extent"], m, cfg["center"], cfg["core_radius"],
                                cfg["edge_scale"], cfg["ppc"], cfg["seed"])
    vel = np.zeros_like(pos)
    work0 = true_work(counts, m, cfg["work_weights"])
    kind = cfg["initial_mapping"]
    if kind == "slab":
        owner = slab_mapping(nb, R)
    elif kind == "roundrobin":
        owner = round_robin_mapping(nb, R)
    elif kind == "knapsack":
        owner = knapsack_assign(work0, R)
    else:
        owner = sfc_assign(work0, curve, R)
    initial_owner = owner.copy()
    comm_face, gather_c, redis_pp, redis_lat = resolve_costs(cfg)
    prov = cfg["provider"]
    overhead = cfg["instrumented_overhead"] if prov == "instrumented" else 1.0
    cols = {k: [] for k in ("step", "eff_before", "eff_after", "adopted",
                            "compute_max", "comm_max", "gather", "redistribute",
                            "walltime", "max_rank_particles", "oom")}
    trace = []
    count_trace = []
    snaps = []
    positions = {}
    adoptions = attempts = 0
    oom = False
    for step in range(cfg["steps"]):
        if step == cfg["kick_step"]:
            vel = kick_velocities(pos, cfg["center"], cfg["kick_speed"],
                                  cfg["kick_drift"], cfg["seed"])
        pos, vel = advance_particles(pos, vel, float(nz), float(nx))
        counts = bin_particles(pos, float(m), nbz, nbx)
        if step + 1 in record_positions_at:
            positions[step + 1] = (pos.copy(), vel.copy())
        if record_counts:
            count_trace.append(counts)
        work = true_work(counts, m, cfg["work_weights"])
        if prov == "heuristic":
            wp, wc = cfg["provider_weights"]
            cost = heuristic_cost(counts, cells, wp, wc)
        else:
            cost = measured_cost(work, cfg["noise"], cfg["seed"], step)
        trace.append(cost)
        e_cur, _ = efficiency_flagged(cost, owner, R)
        attempted = should_attempt(cfg["interval"], cfg["static_step"], step,
                                   cfg["steps"])
        adopted = False
        e_after = e_cur
        prev = owner
        if attempted:
            attempts += 1
            if cfg["strategy"] == "knapsack":
                prop = knapsack_assign(cost, R, cfg["cap_factor"])
            else:
                prop = sfc_assign(cost, curve, R)
            e_prop, _ = efficiency_flagged(cost, prop, R)
            adopted = gate(e_cur, e_prop, cfg["threshold"], cfg["threshold_mode"])
            if adopted:
                owner = prop
                e_after = e_prop
                adoptions += 1
                snaps.append((step, owner.copy()))
        # workload.py:314-363 walltime model
        rank_compute = np.bincount(owner, weights=work, minlength=R)
        compute_max = float(np.max(rank_compute))
        off = owner[fa] != owner[fb]
        pf = (np.bincount(owner[fa][off], minlength=R)
              + np.bincount(owner[fb][off], minlength=R))
        comm_max = float(pf.max()) * comm_face
        gather = gather_c if attempted else 0.0
        redis = 0.0
        if adopted:
            moved = int(counts[owner != prev].sum())
            redis = redis_lat + redis_pp * moved
        occ = np.bincount(owner, weights=counts, minlength=R)
        mrp = int(occ.max())
        is_oom = cfg["capacity"] is not None and mrp > cfg["capacity"]
        compute_max *= overhead
        comm_max *= overhead
        gather *= overhead
        redis *= overhead
        for k, val in (("step", step), ("eff_before", e_cur), ("eff_after", e_after),
                       ("adopted", adopted), ("compute_max", compute_max),
                       ("comm_max", comm_max), ("gather", gather),
                       ("redistribute", redis),
                       ("walltime", compute_max + comm_max + gather + redis),
                       ("max_rank_particles", mrp), ("oom", is_oom)):
            cols[k].append(val)
        if is_oom:
            oom = True
            break
    done = len(cols["step"])
    eff = np.array(cols["eff_after"])
    summary = dict(completed_steps=done,
                   completion_fraction=done / cfg["steps"],
                   total_walltime=float(sum(cols["walltime"])),
                   mean_efficiency=float(eff.mean()) if done else 0.0,
                   adoption_count=adoptions, attempt_count=attempts, oom=oom,
                   final_particles=int(pos.shape[0]))
    out = dict(metrics={k: np.array(v) for k, v in cols.items()},
               cost_trace=np.array(trace), initial_owner=initial_owner,
               snapshots=snaps, summary=summary, final_pos=pos, final_vel=vel)
    if record_counts:
        out["count_trace"] = np.array(count_trace)
    if record_positions_at:
        out["positions"] = positions
    return out


# ----------------------------------------------------------------------------
# 3D extension (config C4) -- PARITY UNPINNED: the reference is 2D only
# (SPEC.md:96).  Same rules carried to a third axis: boxes are
# (bz*nby + by)*nbx + bx; Morton puts axis 0 on bits 0,3,6,...
# ----------------------------------------------------------------------------

def advance_particles_3d(pos, vel, extent):
    new = pos + vel
    alive = np.ones(pos.shape[0], dtype=bool)
    for a in range(3):
        alive &= (new[:, a] >= 0.0) & (new[:, a] < extent[a])
    return np.ascontiguousarray(new[alive]), np.ascontiguousarray(vel[alive])


def bin_particles_3d(pos, box_size, grid):
    b = [np.trunc(pos[:, a] / box_size).astype(np.int64) for a in range(3)]
    ids = (b[0] * grid[1] + b[1]) * grid[2] + b[2]
    return np.bincount(ids, minlength=grid[0] * grid[1] * grid[2]).astype(np.int64)


def morton_order_3d(grid):
    def spread3(v):
        out, s = 0, 0
        while v:
            out |= (v & 1) << (3 * s)
            v >>= 1
            s += 1
        return out
    n0, n1, n2 = grid
    codes = []
    for i in range(n0 * n1 * n2):
        a, b, c = i // (n1 * n2), (i // n2) % n1, i % n2
        codes.append(spread3(a) | (spread3(b) << 1) | (spread3(c) << 2))
    return np.argsort(np.array(codes, dtype=np.int64), kind="stable").astype(np.int64)
