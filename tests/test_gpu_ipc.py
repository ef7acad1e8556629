"""The fused peer-memory exchange across PROCESSES: two ranks on one GPU,
torch.distributed over gloo (CUDA tensors), receive buffers shared with CUDA
IPC handles (lbx_peer_alloc / lbx_peer_open) -- the same mapping path that
NVLink peers use on a multi-GPU node.  Results must equal the
single-process oracle run with ranks = 2."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import lbsim_oracle as O
from tests.dist_util import free_port
from tests.test_dist_gloo import oracle_cfg, sorted_rows

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _rank(rank, world, port, outdir):
    import torch.distributed as dist

    from paper_2104_11385_b200 import scenarios as S
    from paper_2104_11385_b200.parallel import DistributedSimulation, TorchComm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = S.apply_overrides(S.load_spec("mini"), ranks=world, steps=40)
        sim = DistributedSimulation(spec.scenario, spec.policy, spec.build_provider(),
                                    comm=TorchComm(), device="cuda:0", record_counts=True,
                                    exchange="p2p")
        sim.run()
        res = sim.result()
        pos, vel = sim.local_state()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), mode=sim.exchange,
                 cost_trace=res.cost_trace, count_trace=res.count_trace, pos=pos, vel=vel,
                 eff_after=[m.efficiency_after for m in res.metrics], moved=sim.moved)
        sim.close()
    finally:
        dist.destroy_process_group()


def test_p2p_exchange_across_processes(tmp_path):
    world = 2
    mp.spawn(_rank, args=(world, free_port(), str(tmp_path)), nprocs=world)
    cfg, _ = oracle_cfg("mini", world, {"steps": 40})
    ref = O.run_simulation(cfg, record_counts=True)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for o in outs:
        assert str(o["mode"]) == "p2p"
        assert np.array_equal(o["cost_trace"], ref["cost_trace"])
        assert np.array_equal(o["count_trace"], ref["count_trace"])
        assert o["eff_after"].tolist() == ref["metrics"]["eff_after"].tolist()
    got = sorted_rows(np.column_stack([np.concatenate([o["pos"] for o in outs]),
                                       np.concatenate([o["vel"] for o in outs])]))
    want = sorted_rows(np.column_stack([ref["final_pos"], ref["final_vel"]]))
    assert np.array_equal(got, want)
