"""The multi-GPU path over REAL NCCL (torch.distributed backend "nccl"),
world size 1 on the B200 (the box has one GPU): DistributedSimulation with
TorchComm -- NCCL all-reduce of [counts, clock, emigrants], all-to-all of
records, replicated remap -- against the single-process oracle run; plus the
bench's self-launch path (`bench.py --gpus 1 --force-dist` re-executes
itself under torch.distributed.run and runs the NCCL path) and its refusal
of --gpus N on a box with fewer GPUs."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu

WORKER = r'''
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["LBX_ROOT"])
from paper_2104_11385_b200 import scenarios as S
from paper_2104_11385_b200.parallel import DistributedSimulation, TorchComm
base, exchange, out = sys.argv[1], sys.argv[2], sys.argv[3]
kw = json.loads(sys.argv[4])
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:" + os.environ["PORT"],
                        rank=0, world_size=1, device_id=dev)
assert dist.get_backend() == "nccl"
spec = S.apply_overrides(S.load_spec(base), ranks=1, **kw)
sim = DistributedSimulation(spec.scenario, spec.policy, spec.build_provider(),
                            comm=TorchComm(), device=dev, record_counts=True,
                            exchange=exchange)
sim.run()
res = sim.result()
pos, vel = sim.local_state()[:2]
np.savez(out, cost=res.cost_trace, counts=res.count_trace,
         eff=np.array([m.efficiency_before for m in res.metrics]),
         wall=np.array([m.walltime for m in res.metrics]), pos=pos, vel=vel,
         exchange=np.array([sim.exchange]))
sim.close()
dist.destroy_process_group()
'''


def _port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
@pytest.mark.parametrize("base,kw", [("mini", {"steps": 40}),
                                     ("tight-memory", {"steps": 60, "cost": "measured"})])
def test_nccl_world1_matches_oracle(tmp_path, base, kw, exchange):
    from oracle import lbsim_oracle as O
    from tests.test_dist_gloo import oracle_cfg, sorted_rows

    out = tmp_path / "r0.npz"
    env = dict(os.environ, LBX_ROOT=str(ROOT), PORT=str(_port()), NCCL_DEBUG="INFO",
               NCCL_DEBUG_SUBSYS="INIT")
    p = subprocess.run([sys.executable, "-c", WORKER, base, exchange, str(out), json.dumps(kw)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    assert "nranks 1" in (p.stdout + p.stderr).lower()   # NCCL really built a communicator
    cfg, _ = oracle_cfg(base, 1, kw)
    ref = O.run_simulation(cfg, record_counts=True)
    got = np.load(out)
    assert str(got["exchange"][0]) == exchange
    assert np.array_equal(got["cost"], ref["cost_trace"])
    assert np.array_equal(got["counts"], ref["count_trace"])
    assert got["eff"].tolist() == ref["metrics"]["eff_before"].tolist()
    assert got["wall"].tolist() == ref["metrics"]["walltime"].tolist()
    assert np.array_equal(sorted_rows(np.column_stack([got["pos"], got["vel"]])),
                          sorted_rows(np.column_stack([ref["final_pos"], ref["final_vel"]])))


def _bench(*extra, timeout=900):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *extra], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


def test_bench_self_launch_force_dist_runs_nccl_path():
    p = _bench("--gpus", "1", "--force-dist", "--steps", "3", "--warmup", "3",
               "--replicas", "2", "--no-cpu-baseline", "--no-e2e")
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert lines, p.stdout[-2000:]
    line = lines[-1]
    assert line["n_gpus"] == 1 and line["steps"] == 3
    assert "box ownership over 1 GPUs" in line["parallelism"]
    assert line["config"]["ranks"] == 1
    assert "nranks 1" in (p.stdout + p.stderr).lower()


def test_bench_refuses_more_gpus_than_present():
    import torch
    n = torch.cuda.device_count()
    p = _bench("--gpus", str(n + 1), "--steps", "3", "--warmup", "3", "--replicas", "1",
               timeout=300)
    assert p.returncode != 0
    assert "CUDA device" in p.stderr
