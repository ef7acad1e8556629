"""Host LB step (lbx_lb_step) time per step on the C2 box grid, with and
without remap attempts (interval 10 / never), output arrays pre-faulted or
not (argv[1] == "prefault")."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2104_11385_b200 import _lib  # noqa: E402
from paper_2104_11385_b200.workload import sample_blob, sim_config  # noqa: E402

PREFAULT = len(sys.argv) > 1 and sys.argv[1] == "prefault"
KEYS = ("eff_before", "eff_after", "adopted", "attempted", "compute_max", "comm_max", "gather",
        "redistribute", "walltime", "max_rank_particles", "oom", "n_alive", "cost_trace",
        "count_trace", "clock_trace", "owner", "adopt_steps", "adopt_owners")
T, NB = 2000, 900
res = {}
for ranks in (1, 8, 24):
    for interval in (10, 100000):
        for cost in ("heuristic", "gpuclock"):
            spec, sc = bench.c2_spec(ranks, T, cost)
            conf = sim_config(sc, spec.policy, spec.build_provider())
            conf.interval = interval
            own = (np.arange(NB) * ranks // NB).astype(np.int64)
            h = C.c_void_p()
            _lib.check(_lib.lib.lbx_lb_create(C.byref(h), C.byref(conf), _lib.ptr(own)))
            o = {k: np.zeros(T) for k in ("eff_before", "eff_after", "compute_max", "comm_max",
                                          "gather", "redistribute", "walltime")}
            for k in ("adopted", "attempted", "oom"):
                o[k] = np.zeros(T, dtype=np.uint8)
            o["max_rank_particles"] = np.zeros(T, dtype=np.int64)
            o["n_alive"] = np.zeros(T, dtype=np.int64)
            o["cost_trace"] = np.zeros((T, NB))
            o["adopt_steps"] = np.zeros(T, dtype=np.int64)
            o["adopt_owners"] = np.zeros((T, NB), dtype=np.int64)
            if PREFAULT:
                for v in o.values():
                    v.fill(0)
            o["owner"] = own.copy()
            so = _lib.SimOutputs(*(_lib.ptr(o.get(k)) for k in KEYS), None, 0, 0, 0)
            pos = sample_blob(sc)
            counts = np.bincount((pos[:, 0] // 32).astype(int) * 30 + (pos[:, 1] // 32).astype(int),
                                 minlength=NB).astype(np.int64)
            clk = (counts * 100 + np.random.default_rng(0).integers(0, 50, NB)).astype(np.uint64)
            a, hl = C.c_int32(), C.c_int32()
            args = (_lib.ptr(counts), _lib.ptr(clk), int(counts.sum()), C.byref(so), C.byref(a),
                    C.byref(hl))
            f = _lib.lib.lbx_lb_step
            t0 = time.perf_counter()
            for s in range(T):
                f(h, s, *args)
            res[f"r{ranks}_i{interval}_{cost}"] = round(1e6 * (time.perf_counter() - t0) / T, 2)
            _lib.lib.lbx_lb_destroy(h)
print(res)
