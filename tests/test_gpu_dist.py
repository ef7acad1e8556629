"""The multi-GPU path's device kernels (exchange push, partition, group,
unpack, compaction with kick buffers) on a real GPU: `world` ranks run as
threads sharing cuda:0 through parallel.ThreadComm; results must equal the
single-process oracle with ranks = world (metrics, cost trace, mappings,
particle multiset)."""
import json
import threading
from pathlib import Path

import numpy as np
import pytest

from oracle import lbsim_oracle as O
from tests.test_dist_gloo import oracle_cfg, sorted_rows

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def run_threads(base, world, kw, doc, exchange="auto"):
    from paper_2104_11385_b200 import scenarios as S
    from paper_2104_11385_b200.parallel import DeviceEngine, DistributedSimulation, ThreadComm
    shared = ThreadComm.shared(world)
    spec = S.spec_from_dict(doc) if base == "leaky" else S.load_spec(base)
    spec = S.apply_overrides(spec, ranks=world, **kw)
    outs, errs = [None] * world, []
    outs_mode = [None] * world

    def body(r):
        try:
            torch.cuda.set_device(0)
            sim = DistributedSimulation(spec.scenario, spec.policy, spec.build_provider(),
                                        comm=ThreadComm(shared, r), engine_factory=DeviceEngine,
                                        device="cuda:0", record_counts=True,
                                        exchange="auto" if exchange == "auto_expect_nccl"
                                        else exchange)
            outs_mode[r] = sim.exchange
            sim.run()
            outs[r] = (sim.result(), sim.local_state(), sim.moved.copy())
            sim.close()
        except Exception as e:  # surface in the main thread
            errs.append(e)
            shared["bar"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    want = "nccl" if exchange in ("nccl", "auto_expect_nccl") else "p2p"
    assert all(m == want for m in outs_mode), outs_mode
    return outs


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
@pytest.mark.parametrize("base,world,kw", [("mini", 2, {"steps": 40}),
                                           ("mini", 3, {"steps": 40, "policy": "sfc"}),
                                           ("leaky", 3, {}),
                                           ("tight-memory", 2, {"steps": 60, "cost": "measured"})])
def test_gpu_distributed_matches_oracle(base, world, kw, exchange):
    """exchange='p2p': the fused push + exchange writes emigrants straight
    into the destination rank's receive buffer (peer memory; here the ranks
    share one GPU); 'nccl': staged records + all-to-all collectives."""
    cfg, doc = oracle_cfg(base, world, kw)
    outs = run_threads(base, world, kw, doc, exchange)
    ref = O.run_simulation(cfg, record_counts=True)
    for res, _, _ in outs:
        m = res.metrics
        assert [x.efficiency_before for x in m] == ref["metrics"]["eff_before"].tolist()
        assert [x.adopted for x in m] == ref["metrics"]["adopted"].tolist()
        assert [x.walltime for x in m] == ref["metrics"]["walltime"].tolist()
        assert np.array_equal(res.cost_trace, ref["cost_trace"])
        assert np.array_equal(res.count_trace, ref["count_trace"])
        assert [s for s, _ in res.adoption_snapshots] == [s for s, _ in ref["snapshots"]]
    pos = np.concatenate([st[0] for _, st, _ in outs])
    vel = np.concatenate([st[1] for _, st, _ in outs])
    assert np.array_equal(sorted_rows(np.column_stack([pos, vel])),
                          sorted_rows(np.column_stack([ref["final_pos"], ref["final_vel"]])))
    if any(ref["metrics"]["adopted"]):
        assert sum(mv.sum() for _, _, mv in outs) > 0


def test_gpu_distributed_gpuclock_runs():
    """GpuClock costs across ranks: every rank's clock tally is all-reduced,
    so all ranks see the same cost vector and take the same decisions."""
    cfg, doc = oracle_cfg("mini", 2, {"steps": 30})
    outs = run_threads("mini", 2, {"steps": 30, "cost": "gpuclock"}, doc)
    a, b = outs[0][0], outs[1][0]
    assert np.array_equal(a.cost_trace, b.cost_trace)
    assert [m.adopted for m in a.metrics] == [m.adopted for m in b.metrics]
    ref = O.run_simulation(cfg, record_counts=True)
    assert np.array_equal(a.count_trace, ref["count_trace"])
    # calibrated GpuClock: clock share + the per-box cell work w_c M^2
    cell = 0.25 * float(cfg["box_size"] ** 2)
    assert ((a.cost_trace > cell) == (ref["count_trace"] > 0)).all()


@pytest.mark.parametrize("world", [2, 3])
def test_gpu_distributed_pic_matches_oracle(world):
    """parallel.PicEngine on the GPU, ranks as threads: libLBX PIC step with
    the current deferred, guard-cell exchange of the integer current rows
    along shared faces, lbx_pic_finish over the rank's region, guard-ring
    field exchange, emigrant exchange and adoption-time migration (+ field
    sync to the new owners) -- bit-identical to the single-process oracle
    PIC run on every rank's own cells."""
    from paper_2104_11385_b200 import scenarios as S
    from paper_2104_11385_b200.parallel import DistributedSimulation, ThreadComm
    from tests.dist_util import pic_reference
    doc = json.loads((Path(__file__).parent / "golden" / "runs.json").read_text())["_docs"]["small"]
    steps = 16
    spec = S.apply_overrides(S.spec_from_dict(doc), ranks=world, steps=steps, interval=3,
                             threshold=0.0)
    shared = ThreadComm.shared(world)
    outs, errs = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            sim = DistributedSimulation(spec.scenario, spec.policy, spec.build_provider(),
                                        comm=ThreadComm(shared, r), device="cuda:0",
                                        record_counts=True, physics="pic")
            sim.run()
            outs[r] = (sim.result(), sim.engine.state(), sim.engine.field_arrays(),
                       sim.moved.copy(), sim.engine.halo.owner.copy(),
                       sim.engine.halo.bytes_j + sim.engine.halo.bytes_f)
            sim.close()
        except Exception as e:
            errs.append(e)
            shared["bar"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    from tests.dist_util import own_cells_mask
    counts, p, f = pic_reference(doc, steps)
    keys = ("z", "x", "uz", "ux", "uy")
    nz, nx = doc["domain"]["extent"]
    box = doc["domain"]["box_size"]
    cover = np.zeros((nz + 2, nx + 2), dtype=bool)
    for r, (res, _, fa, _, owner, nbytes) in enumerate(outs):
        assert np.array_equal(res.count_trace, counts)
        mine = own_cells_mask(owner, ((nz // box, nx // box), box, nz, nx), r)
        cover |= mine
        for k in ("Ex", "Ey", "Ez", "Bx", "By", "Bz"):
            assert np.array_equal(fa[k][mine], f[k][mine]), (r, k)
        # guard exchange: far less than the replicated current (16 int64 per cell)
        assert 0 < nbytes < 16 * 8 * nz * nx
    assert cover[1:-1, 1:-1].all()
    got = sorted_rows(np.column_stack([np.concatenate([o[1][k] for o in outs]) for k in keys]))
    want = sorted_rows(np.column_stack([p[k] for k in keys]))
    assert np.array_equal(got, want)
    assert outs[0][0].summary["adoption_count"] > 0 and sum(o[3].sum() for o in outs) > 0


@pytest.mark.parametrize("world", [2, 3])
def test_gpu_distributed_pic_esirkepov(world):
    """Distributed PIC with the paper's order-3 charge-conserving deposition
    (shape_order 3, ranks cell-sort their particles every 4 steps): each rank defers its node-centric Esirkepov sums, the
    sums near shared faces are exchanged and added (PicHalo order 3), every
    rank finishes its region and the guard rings (3 cells) come from their
    owners.  Against the single-process oracle Esirkepov run (tolerance
    mode): per-box counts exact, fields on every rank's own cells and the
    particle multiset within tests/test_gpu_pic_esirkepov.py's tolerances."""
    from paper_2104_11385_b200 import scenarios as S
    from paper_2104_11385_b200.parallel import DistributedSimulation, ThreadComm
    from tests.dist_util import own_cells_mask, pic_reference
    from tests.test_gpu_pic_esirkepov import F_TOL, U_TOL, X_TOL
    doc = json.loads((Path(__file__).parent / "golden" / "runs.json").read_text())["_docs"]["small"]
    steps = 12
    spec = S.apply_overrides(S.spec_from_dict(doc), ranks=world, steps=steps, interval=3,
                             threshold=0.0)
    shared = ThreadComm.shared(world)
    outs, errs = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            sim = DistributedSimulation(spec.scenario, spec.policy, spec.build_provider(),
                                        comm=ThreadComm(shared, r), device="cuda:0",
                                        record_counts=True, physics="pic",
                                        pic={"shape_order": 3, "resort": 4})
            sim.run()
            assert sim.engine.order == 3 and sim.engine.halo.guard == 3
            outs[r] = (sim.result(), sim.engine.state(), sim.engine.field_arrays(),
                       sim.engine.halo.owner.copy(), sim.engine.halo.bytes_j)
            sim.close()
        except Exception as e:
            errs.append(e)
            shared["bar"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    counts, p, f = pic_reference(doc, steps, order=3)
    nz, nx = doc["domain"]["extent"]
    box = doc["domain"]["box_size"]
    for r, (res, _, fa, owner, nbytes) in enumerate(outs):
        assert np.array_equal(res.count_trace, counts)
        mine = own_cells_mask(owner, ((nz // box, nx // box), box, nz, nx), r)
        for k in ("Ex", "Ey", "Ez", "Bx", "By", "Bz"):
            scale = max(float(np.abs(f[k]).max()), 1e-30)
            assert np.abs(fa[k][mine] - f[k][mine]).max() / scale <= F_TOL, (r, k)
        assert 0 < nbytes < 3 * 8 * nz * nx
    umax = max(float(np.abs(p[k]).max()) for k in ("uz", "ux", "uy"))
    for k, tol in (("z", X_TOL), ("x", X_TOL), ("uz", U_TOL * umax), ("ux", U_TOL * umax),
                   ("uy", U_TOL * umax)):
        got = np.sort(np.concatenate([o[1][k] for o in outs]))
        assert got.shape == p[k].shape
        assert np.abs(got - np.sort(p[k])).max() <= tol, k
    assert outs[0][0].summary["adoption_count"] > 0


def test_gpu_distributed_pic_tolerance_mode():
    """Distributed PIC in tolerance mode (pic={"fast": True}: LBX_PIC_FAST,
    the pipelined kernel where the quad copy pays) on 2 thread ranks with the
    current deferred and the face-band exchange: per-box counts exact, the
    particle multiset and the fields of every rank's own cells within
    tests/test_gpu_pic_fast.py's tolerances of the single-process oracle."""
    from paper_2104_11385_b200 import scenarios as S
    from paper_2104_11385_b200.parallel import DistributedSimulation, ThreadComm
    from tests.dist_util import own_cells_mask, pic_reference
    from tests.test_gpu_pic_fast import F_TOL, U_TOL, X_TOL
    doc = json.loads((Path(__file__).parent / "golden" / "runs.json").read_text())["_docs"]["small"]
    steps, world = 12, 2
    spec = S.apply_overrides(S.spec_from_dict(doc), ranks=world, steps=steps, interval=3,
                             threshold=0.0)
    shared = ThreadComm.shared(world)
    outs, errs = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            sim = DistributedSimulation(spec.scenario, spec.policy, spec.build_provider(),
                                        comm=ThreadComm(shared, r), device="cuda:0",
                                        record_counts=True, physics="pic",
                                        pic={"fast": True, "resort": 4})
            sim.run()
            assert sim.engine.fast
            outs[r] = (sim.result(), sim.engine.state(), sim.engine.field_arrays(),
                       sim.engine.halo.owner.copy())
            sim.close()
        except Exception as e:
            errs.append(e)
            shared["bar"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    counts, p, f = pic_reference(doc, steps)
    nz, nx = doc["domain"]["extent"]
    box = doc["domain"]["box_size"]
    for r, (res, _, fa, owner) in enumerate(outs):
        assert np.array_equal(res.count_trace, counts)
        mine = own_cells_mask(owner, ((nz // box, nx // box), box, nz, nx), r)
        for k in ("Ex", "Ey", "Ez", "Bx", "By", "Bz"):
            scale = max(float(np.abs(f[k]).max()), 1e-30)
            assert np.abs(fa[k][mine] - f[k][mine]).max() / scale <= F_TOL, (r, k)
    umax = max(float(np.abs(p[k]).max()) for k in ("uz", "ux", "uy"))
    for k, tol in (("z", X_TOL), ("x", X_TOL), ("uz", U_TOL * umax), ("ux", U_TOL * umax),
                   ("uy", U_TOL * umax)):
        got = np.sort(np.concatenate([o[1][k] for o in outs]))
        assert np.abs(got - np.sort(p[k])).max() <= tol, k


def test_p2p_failure_on_one_rank_falls_back_to_collectives(monkeypatch):
    """If any rank cannot map peer memory, every rank switches to the
    collective exchange together and the run stays exact."""
    from paper_2104_11385_b200.parallel import DeviceEngine
    orig = DeviceEngine.p2p_alloc

    def flaky(self):
        if self.rank == 1:
            raise RuntimeError("simulated peer-buffer failure")
        return orig(self)

    monkeypatch.setattr(DeviceEngine, "p2p_alloc", flaky)
    cfg, doc = oracle_cfg("mini", 2, {"steps": 30})
    outs = run_threads("mini", 2, {"steps": 30}, doc, exchange="auto_expect_nccl")
    ref = O.run_simulation(cfg, record_counts=True)
    for res, _, _ in outs:
        assert np.array_equal(res.cost_trace, ref["cost_trace"])
        assert np.array_equal(res.count_trace, ref["count_trace"])


def test_measured_migration_prices_the_gate():
    """policy.measured_migration: every adoption's redistribution is timed
    (max over ranks) against the push, the per-particle price is fed to the
    native gate (lbx_lb_set_migration_ratio) identically on every rank, and
    later adoptions must save more load than the measured move costs -- so
    there are at most as many adoptions as with the reference gate."""
    from dataclasses import replace

    from paper_2104_11385_b200 import scenarios as S
    from paper_2104_11385_b200.parallel import DistributedSimulation, ThreadComm
    world = 2
    res = {}
    for measured in (False, True):
        spec = S.apply_overrides(S.load_spec("mini"), ranks=world, steps=60, interval=3,
                                 threshold=0.0)
        policy = replace(spec.policy, measured_migration=measured)
        shared = ThreadComm.shared(world)
        outs, errs = [None] * world, []

        def body(r):
            try:
                torch.cuda.set_device(0)
                sim = DistributedSimulation(spec.scenario, policy, spec.build_provider(),
                                            comm=ThreadComm(shared, r), device="cuda:0")
                sim.run()
                outs[r] = (sim.result(), list(sim.mig_log), sim.mig_ratio)
                sim.close()
            except Exception as e:
                errs.append(e)
                shared["bar"].abort()

        th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        a, b = outs
        assert [m.adopted for m in a[0].metrics] == [m.adopted for m in b[0].metrics]
        assert a[1] == b[1] and a[2] == b[2]      # same measurements, same price
        res[measured] = outs[0]
    base, meas = res[False], res[True]
    assert meas[1], "no adoption was measured"
    assert all(x["migration_ms"] > 0 and x["push_ms"] > 0 for x in meas[1])
    assert meas[2] > 0
    assert meas[0].summary["adoption_count"] <= base[0].summary["adoption_count"]
