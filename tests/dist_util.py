"""Test double for parallel.DeviceEngine: the same per-rank operations in
numpy on CPU tensors, built from the oracle's kernels, so the distributed
protocol (collectives, exchange bookkeeping, replicated LB) can be tested
with gloo on a machine without a GPU."""
import os
import socket

import numpy as np
import torch

from oracle import lbsim_oracle as O

REC = 6


class NumpyEngine:
    def __init__(self, cfg, rank, world, device, pos, kick, capacity, clock):
        self.rank, self.world = rank, world
        self.ez, self.ex = float(cfg.domain_extent[0]), float(cfg.domain_extent[1])
        self.m = float(cfg.box_size)
        self.nbz, self.nbx = cfg.domain_extent[0] // cfg.box_size, cfg.domain_extent[1] // cfg.box_size
        self.pos = np.array(pos, dtype=np.float64).reshape(-1, 2)
        self.vel = np.zeros_like(self.pos)
        self.kick_v = None if kick is None else np.array(kick, dtype=np.float64).reshape(-1, 2)
        self.owner = None
        self.staged = np.zeros((0, REC))
        self.dest = np.zeros(0, dtype=np.int64)

    @property
    def n(self):
        return self.pos.shape[0]

    def set_owner(self, owner):
        self.owner = np.asarray(owner, dtype=np.int64)

    def kick(self):
        if self.kick_v is not None:
            self.vel, self.kick_v = self.kick_v, None

    def _records(self, idx, pos):
        k = self.kick_v[idx] if self.kick_v is not None else np.zeros((idx.size, 2))
        return np.column_stack([pos[idx], self.vel[idx], k])

    def _split(self, pos, alive):
        box = np.full(pos.shape[0], -1, dtype=np.int64)
        box[alive] = (np.trunc(pos[alive, 0] / self.m).astype(np.int64) * self.nbx
                      + np.trunc(pos[alive, 1] / self.m).astype(np.int64))
        emig = np.zeros(pos.shape[0], dtype=bool)
        emig[alive] = self.owner[box[alive]] != self.rank
        idx = np.flatnonzero(emig)
        self.staged = self._records(idx, pos)
        self.dest = self.owner[box[idx]]
        stay = alive & ~emig
        self.pos, self.vel = pos[stay], self.vel[stay]
        if self.kick_v is not None:
            self.kick_v = self.kick_v[stay]
        return box, alive

    def push(self, wp, wc):
        pos = self.pos + self.vel
        alive = ((pos[:, 0] >= 0) & (pos[:, 0] < self.ez) & (pos[:, 1] >= 0)
                 & (pos[:, 1] < self.ex))
        box, alive = self._split(pos, alive)
        counts = np.bincount(box[alive], minlength=self.nbz * self.nbx).astype(np.int64)
        send = np.bincount(self.dest, minlength=self.world).astype(np.int64)
        return (torch.from_numpy(counts), torch.zeros(counts.size, dtype=torch.int64),
                torch.from_numpy(send), torch.tensor([self.n, 0], dtype=torch.int64))

    def partition(self):
        self._split(self.pos.copy(), np.ones(self.n, dtype=bool))
        return (torch.from_numpy(np.bincount(self.dest, minlength=self.world).astype(np.int64)),
                torch.tensor([self.n, 0], dtype=torch.int64))

    def commit(self, nout_host):
        assert int(nout_host[0]) == self.n

    def pack(self, sc):
        order = np.argsort(self.dest, kind="stable")
        return torch.from_numpy(np.ascontiguousarray(self.staged[order]).reshape(-1, REC))

    def unpack(self, recv):
        r = recv.numpy().reshape(-1, REC)
        self.pos = np.concatenate([self.pos, r[:, 0:2]])
        self.vel = np.concatenate([self.vel, r[:, 2:4]])
        if self.kick_v is not None:
            self.kick_v = np.concatenate([self.kick_v, r[:, 4:6]])

    def state(self):
        return self.pos.copy(), self.vel.copy()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_rank(rank, world, port, spec_kw, outdir, engine="numpy"):
    """mp.spawn target: one gloo rank of a DistributedSimulation."""
    import torch.distributed as dist

    from paper_2104_11385_b200 import scenarios as S
    from paper_2104_11385_b200.parallel import DistributedSimulation, TorchComm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        base = spec_kw.pop("_base")
        spec = S.spec_from_dict(base) if isinstance(base, dict) else S.load_spec(base)
        spec = S.apply_overrides(spec, ranks=world, **spec_kw)
        sim = DistributedSimulation(spec.scenario, spec.policy, spec.build_provider(),
                                    comm=TorchComm(), engine_factory=NumpyEngine,
                                    record_counts=True)
        sim.run()
        res = sim.result()
        pos, vel = sim.local_state()
        m = res.metrics
        np.savez(os.path.join(outdir, f"rank{rank}.npz"),
                 eff_before=[x.efficiency_before for x in m],
                 eff_after=[x.efficiency_after for x in m],
                 adopted=[x.adopted for x in m], walltime=[x.walltime for x in m],
                 compute_max=[x.compute_max for x in m], comm_max=[x.comm_max for x in m],
                 redistribute=[x.redistribute for x in m],
                 mrp=[x.max_rank_particles for x in m], oom=[x.oom for x in m],
                 cost_trace=res.cost_trace, count_trace=res.count_trace,
                 initial_owner=res.initial_owner, pos=pos, vel=vel,
                 snap_steps=[s for s, _ in res.adoption_snapshots],
                 snap_owner=np.array([o for _, o in res.adoption_snapshots]).reshape(
                     -1, res.initial_owner.size),
                 moved=sim.moved, mean_eff=res.summary["mean_efficiency"],
                 completed=res.summary["completed_steps"])
        sim.close()
    finally:
        dist.destroy_process_group()


class NumpyPicEngine:
    """Test double for parallel.PicEngine: the same per-rank PIC protocol in
    numpy (oracle/pic_oracle.py) -- push the local particles, exchange the
    integer node current of the cells along shared faces (parallel.halo_plan:
    node sums of the cells within two cells of the sender's boxes that the
    receiver owns), apply it and run the field solve, exchange the owners'
    E, B values of the two-cell guard rings, then stage emigrants as
    6-double records.  Each rank's fields are current on its own cells."""

    def __init__(self, cfg, rank, world, device, pos, kick, capacity, clock, pic=None):
        from oracle import pic_oracle as PO
        from paper_2104_11385_b200.workload import PIC_DEFAULTS
        self.PO = PO
        self.pic = dict(PIC_DEFAULTS, **(pic or {}))
        self.rank, self.world = rank, world
        self.nz, self.nx = cfg.domain_extent
        self.m = float(cfg.box_size)
        self.nbz, self.nbx = self.nz // cfg.box_size, self.nx // cfg.box_size
        pos = np.array(pos, dtype=np.float64).reshape(-1, 2)
        z0 = np.zeros(pos.shape[0])
        self.p = {"z": pos[:, 0].copy(), "x": pos[:, 1].copy(), "uz": z0.copy(),
                  "ux": z0.copy(), "uy": z0.copy()}
        self.kick_v = None if kick is None else np.array(kick, dtype=np.float64).reshape(-1, 2)
        self.f = PO.new_fields(self.nz, self.nx)
        self.owner = None
        self.staged = np.zeros((0, REC))
        self.dest = np.zeros(0, dtype=np.int64)
        self.comm = None

    @property
    def n(self):
        return self.p["z"].size

    def attach_comm(self, comm):
        self.comm = comm

    def set_owner(self, owner):
        from paper_2104_11385_b200.parallel import cell_owner_map, halo_plan
        owner = np.asarray(owner, dtype=np.int64)
        grid = (self.nbz, self.nbx)
        new = cell_owner_map(owner, grid, int(self.m))
        if self.owner is not None and not np.array_equal(owner, self.owner):
            old = cell_owner_map(self.owner, grid, int(self.m))
            self._fields_exchange(*halo_plan(old, new, self.rank, self.world, 0, 2))
        self.owner = owner
        self.j_plan = halo_plan(new, new, self.rank, self.world, 2, 0)
        self.f_plan = halo_plan(new, new, self.rank, self.world, 0, 2)

    def _exchange(self, arrays, plan):
        """Interior (cell) values of `arrays` at plan's send cells -> peers;
        returns (received (m, k) values, the cells they belong to)."""
        send_idx, recv_idx = plan
        send = np.concatenate([np.column_stack([a.reshape(-1)[self._pad(ix)] for a in arrays])
                               for ix in send_idx]) if sum(map(len, send_idx)) else \
            np.zeros((0, len(arrays)), dtype=arrays[0].dtype)
        k = len(arrays)
        t = torch.from_numpy(np.ascontiguousarray(send).reshape(-1))
        r = self.comm.exchange_values(t, [k * len(ix) for ix in send_idx],
                                      [k * len(ix) for ix in recv_idx])
        return r.numpy().reshape(-1, k), self._pad(np.concatenate(recv_idx))

    def _pad(self, cells):
        """flat cell index -> flat index of its node in the padded arrays"""
        return (cells // self.nx + 1) * (self.nx + 2) + (cells % self.nx + 1)

    def _fields_exchange(self, send_idx, recv_idx):
        names = self.PO.E_COMPS + self.PO.B_COMPS
        vals, cells = self._exchange([self.f[k] for k in names], (send_idx, recv_idx))
        for c, k in enumerate(names):
            self.f[k].reshape(-1)[cells] = vals[:, c]

    def kick(self):
        if self.kick_v is not None:
            self.p["uz"] = self.kick_v[:, 0] / self.pic["dt"]
            self.p["ux"] = self.kick_v[:, 1] / self.pic["dt"]
            self.kick_v = None

    def _records(self, idx):
        p = self.p
        tail = (self.kick_v[idx] if self.kick_v is not None
                else np.column_stack([p["uy"][idx], np.zeros(idx.size)]))
        return np.column_stack([p["z"][idx], p["x"][idx], p["uz"][idx], p["ux"][idx], tail])

    def _split(self):
        p = self.p
        box = (np.trunc(p["z"] / self.m).astype(np.int64) * self.nbx
               + np.trunc(p["x"] / self.m).astype(np.int64))
        emig = self.owner[box] != self.rank
        idx = np.flatnonzero(emig)
        self.staged = self._records(idx)
        self.dest = self.owner[box[idx]]
        stay = ~emig
        self.p = {k: v[stay] for k, v in p.items()}
        if self.kick_v is not None:
            self.kick_v = self.kick_v[stay]
        return box[stay]

    def push(self, wp, wc):
        PO, c = self.PO, self.pic
        keep, ig = PO.push_particles(self.f, self.p, self.nz, self.nx, c["q_over_m"], c["dt"])
        if self.kick_v is not None:
            self.kick_v = self.kick_v[keep]
        box = (np.trunc(self.p["z"] / self.m).astype(np.int64) * self.nbx
               + np.trunc(self.p["x"] / self.m).astype(np.int64))
        counts = np.bincount(box, minlength=self.nbz * self.nbx).astype(np.int64)
        shape = self.f["Jx"].shape
        sc = PO.current_scale(c["q_times_w"])
        accs = PO.current_accs(self.p, ig, c["q_times_w"], shape)
        comps = ("Jx", "Jy", "Jz")
        vals, cells = self._exchange([accs[k] for k in comps], self.j_plan)
        for i, k in enumerate(comps):
            np.add.at(accs[k].reshape(-1), cells, vals[:, i])
            PO.apply_current(self.f, k, accs[k], sc)
        PO.field_step(self.f, self.nz, self.nx, c["dt"])
        self._fields_exchange(*self.f_plan)
        self._split()
        send = np.bincount(self.dest, minlength=self.world).astype(np.int64)
        return (torch.from_numpy(counts), torch.zeros(counts.size, dtype=torch.int64),
                torch.from_numpy(send), torch.tensor([self.n, 0], dtype=torch.int64))

    def partition(self):
        self._split()
        return (torch.from_numpy(np.bincount(self.dest, minlength=self.world).astype(np.int64)),
                torch.tensor([self.n, 0], dtype=torch.int64))

    def commit(self, nout_host):
        assert int(nout_host[0]) == self.n

    def pack(self, sc):
        order = np.argsort(self.dest, kind="stable")
        return torch.from_numpy(np.ascontiguousarray(self.staged[order]).reshape(-1, REC))

    def unpack(self, recv):
        r = recv.numpy().reshape(-1, REC)
        add = {"z": r[:, 0], "x": r[:, 1], "uz": r[:, 2], "ux": r[:, 3],
               "uy": r[:, 4] if self.kick_v is None else np.zeros(r.shape[0])}
        self.p = {k: np.concatenate([self.p[k], add[k]]) for k in self.p}
        if self.kick_v is not None:
            self.kick_v = np.concatenate([self.kick_v, r[:, 4:6]])

    def state(self):
        return {k: v.copy() for k, v in self.p.items()}

    def field_arrays(self):
        return {k: v.copy() for k, v in self.f.items()}


def pic_reference(doc, steps, order=0):
    """Single-process oracle PIC run of a scenario doc (kick -> u = v/dt):
    per-step per-box counts, final particles and fields.  order > 0: the
    Esirkepov step with B-spline shapes of that order."""
    from oracle import lbsim_oracle as LO
    from oracle import pic_oracle as PO
    from paper_2104_11385_b200 import scenarios as S
    from paper_2104_11385_b200.workload import PIC_DEFAULTS, kick_velocities, sample_blob
    spec = S.apply_overrides(S.spec_from_dict(doc), steps=steps)
    cfg = spec.scenario
    c = PIC_DEFAULTS
    pos = sample_blob(cfg)
    kick = kick_velocities(pos, cfg)
    nz, nx = cfg.domain_extent
    f = PO.new_fields(nz, nx)
    z0 = np.zeros(len(pos))
    p = {"z": pos[:, 0].copy(), "x": pos[:, 1].copy(), "uz": z0.copy(), "ux": z0.copy(),
         "uy": z0.copy()}
    counts = []
    for step in range(cfg.total_steps):
        if step == cfg.kick.step:
            p["uz"], p["ux"] = kick[:, 0] / c["dt"], kick[:, 1] / c["dt"]
        if order:
            PO.particle_step_esirkepov(f, p, nz, nx, c["q_over_m"], c["q_times_w"], c["dt"], order)
        else:
            PO.particle_step(f, p, nz, nx, c["q_over_m"], c["q_times_w"], c["dt"])
        PO.field_step(f, nz, nx, c["dt"])
        counts.append(LO.bin_particles(np.column_stack([p["z"], p["x"]]), float(cfg.box_size),
                                       nz // cfg.box_size, nx // cfg.box_size))
    return np.array(counts), p, f


def run_rank_pic(rank, world, port, doc, steps, outdir, overrides=None):
    """mp.spawn target: one gloo rank of a distributed PIC run."""
    import torch.distributed as dist

    from paper_2104_11385_b200 import scenarios as S
    from paper_2104_11385_b200.parallel import DistributedSimulation, TorchComm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = S.apply_overrides(S.spec_from_dict(doc), ranks=world, steps=steps,
                                 **(overrides or {}))
        sim = DistributedSimulation(spec.scenario, spec.policy, spec.build_provider(),
                                    comm=TorchComm(), engine_factory=NumpyPicEngine,
                                    record_counts=True, physics="pic")
        sim.run()
        res = sim.result()
        st = sim.engine.state()
        f = sim.engine.field_arrays()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), count_trace=res.count_trace,
                 adoptions=res.summary["adoption_count"], moved=sim.moved,
                 owner=np.asarray(sim.engine.owner),
                 **{f"p_{k}": v for k, v in st.items()}, **{f"f_{k}": v for k, v in f.items()})
        sim.close()
    finally:
        dist.destroy_process_group()


def own_cells_mask(owner, cfg_doc_or_shape, rank):
    """Boolean (nz + 2, nx + 2) mask of the padded field nodes of `rank`'s cells."""
    from paper_2104_11385_b200.parallel import cell_owner_map
    grid, box, nz, nx = cfg_doc_or_shape
    cells = cell_owner_map(owner, grid, box) == rank
    m = np.zeros((nz + 2, nx + 2), dtype=bool)
    m[1:-1, 1:-1] = cells
    return m
