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
