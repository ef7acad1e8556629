"""Test double for three_d.Engine3D: the same per-rank 3D operations in numpy
(the oracle's 3D push / bin rules), so Distributed3D's protocol -- global
counts by all-reduce, emigrant exchange, replicated LB, adoption-time
migration -- runs with gloo on a machine without a GPU."""
import os

import numpy as np
import torch

from oracle import lbsim_oracle as O

REC3 = 6


class NumpyEngine3D:
    def __init__(self, cfg, rank, world, device, pos, kick, capacity, clock):
        self.cfg, self.rank, self.world = cfg, rank, world
        self.pos = np.array(pos, dtype=np.float64).reshape(-1, 3)
        self.vel = np.zeros_like(self.pos)
        self.pending = None if kick is None else np.array(kick, dtype=np.float64).reshape(-1, 3)
        self.owner = None
        self.staged = np.zeros((0, REC3))
        self.dest = np.zeros(0, dtype=np.int64)

    @property
    def n(self):
        return self.pos.shape[0]

    def set_owner(self, owner):
        self.owner = np.asarray(owner, dtype=np.int64)

    def kick(self):
        if self.pending is not None:
            self.vel, self.pending = self.pending, None

    def _box(self, pos):
        g = self.cfg.grid
        b = np.trunc(pos / self.cfg.box_size).astype(np.int64)
        return (b[:, 0] * g[1] + b[:, 1]) * g[2] + b[:, 2]

    def _split(self, pos, vel, alive):
        box = np.full(pos.shape[0], -1, dtype=np.int64)
        box[alive] = self._box(pos[alive])
        emig = np.zeros(pos.shape[0], dtype=bool)
        emig[alive] = self.owner[box[alive]] != self.rank
        idx = np.flatnonzero(emig)
        carry = vel if self.pending is None else self.pending
        self.staged = np.column_stack([pos[idx], carry[idx]])
        self.dest = self.owner[box[idx]]
        stay = alive & ~emig
        self.pos, self.vel = pos[stay], vel[stay]
        if self.pending is not None:
            self.pending = self.pending[stay]
        return box

    def push(self, wp, wc):
        pos = self.pos + self.vel
        ext = self.cfg.domain_extent
        alive = np.ones(pos.shape[0], dtype=bool)
        for a in range(3):
            alive &= (pos[:, a] >= 0.0) & (pos[:, a] < ext[a])
        box = self._split(pos, self.vel, alive)
        counts = np.bincount(box[alive], minlength=self.cfg.n_boxes).astype(np.int64)
        send = np.bincount(self.dest, minlength=self.world).astype(np.int64)
        return (torch.from_numpy(counts), torch.zeros(counts.size, dtype=torch.int64),
                torch.from_numpy(send), torch.tensor([self.n, 0], dtype=torch.int64))

    def partition(self):
        self._split(self.pos.copy(), self.vel.copy(), np.ones(self.n, dtype=bool))
        return (torch.from_numpy(np.bincount(self.dest, minlength=self.world).astype(np.int64)),
                torch.tensor([self.n, 0], dtype=torch.int64))

    def commit(self, nout_host):
        assert int(nout_host[0]) == self.n

    def pack(self, sc):
        order = np.argsort(self.dest, kind="stable")
        return torch.from_numpy(np.ascontiguousarray(self.staged[order]).reshape(-1, REC3))

    def unpack(self, recv):
        r = recv.numpy().reshape(-1, REC3)
        self.pos = np.concatenate([self.pos, r[:, 0:3]])
        if self.pending is None:
            self.vel = np.concatenate([self.vel, r[:, 3:6]])
        else:
            self.vel = np.concatenate([self.vel, np.zeros((r.shape[0], 3))])
            self.pending = np.concatenate([self.pending, r[:, 3:6]])

    def state(self):
        return self.pos.copy(), self.vel.copy()


def run_rank3d(rank, world, port, cfg_kw, pol_kw, outdir):
    """mp.spawn target: one gloo rank of a Distributed3D run."""
    import torch.distributed as dist

    from paper_2104_11385_b200.balancer import BalancePolicy, Strategy
    from paper_2104_11385_b200.cost import make_provider
    from paper_2104_11385_b200.parallel import TorchComm
    from paper_2104_11385_b200.three_d import Distributed3D, Scenario3D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = Scenario3D(**cfg_kw)
        pol = BalancePolicy(strategy=Strategy(pol_kw["strategy"]), interval=pol_kw["interval"])
        sim = Distributed3D(cfg, pol, make_provider("heuristic"), comm=TorchComm(),
                            engine_factory=NumpyEngine3D, record_counts=True)
        sim.run()
        pos, vel = sim.local_state()
        o = sim.out
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), count_trace=o["count_trace"],
                 cost_trace=o["cost_trace"], eff_before=o["eff_before"],
                 eff_after=o["eff_after"], adopted=o["adopted"], walltime=o["walltime"],
                 adopt_owners=o["adopt_owners"][:int(sim.souts.n_adoptions)],
                 pos=pos, vel=vel, moved=sim.moved)
        sim.close()
    finally:
        dist.destroy_process_group()
