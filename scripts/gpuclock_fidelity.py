"""GpuClock fidelity at the reference's own C2 size:
default.yaml (801,499 particles, 900 boxes, 24 ranks, 2000 steps) through
the native loop with each cost strategy; reports mean E on the strategy's
own costs, mean E of its mappings under TRUE work, adoptions, and the
Spearman correlation of the clock tally with the particle counts."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import lbsim_oracle as O  # noqa: E402
from paper_2104_11385_b200 import scenarios as S  # noqa: E402
from paper_2104_11385_b200.workload import run_simulation  # noqa: E402


def true_eff(res, cfg):
    owner = res.initial_owner.copy()
    snaps = dict((s, o) for s, o in res.adoption_snapshots)
    effs = []
    for s in range(res.count_trace.shape[0]):
        if s in snaps:
            owner = snaps[s]
        work = O.true_work(res.count_trace[s], cfg.box_size, cfg.work_weights)
        effs.append(O.efficiency_flagged(work, owner, cfg.n_ranks)[0])
    return np.array(effs)


def main(preset="default", ranks=None):
    out = {"preset": preset}
    for kind in ("heuristic", "measured", "gpuclock", "gpuclock-raw"):
        kw = {"cost": kind}
        if ranks:
            kw["ranks"] = ranks
        spec = S.apply_overrides(S.load_spec(preset), **kw)
        t0 = time.perf_counter()
        res = run_simulation(spec.scenario, spec.policy, spec.build_provider(),
                             record_counts=True, record_clock=kind.startswith("gpuclock"))
        el = time.perf_counter() - t0
        te = true_eff(res, spec.scenario)
        d = {"mean_E_own_costs": res.summary["mean_efficiency"],
             "mean_E_true_work": float(te.mean()), "adoptions": res.summary["adoption_count"],
             "seconds": el, "ranks": spec.scenario.n_ranks}
        if res.clock_trace is not None:
            rhos = []
            for s in range(0, spec.scenario.total_steps, 10):
                occ = res.count_trace[s] > 0
                rc = np.argsort(np.argsort(res.clock_trace[s][occ]))
                rw = np.argsort(np.argsort(res.count_trace[s][occ]))
                rhos.append(float(np.corrcoef(rc, rw)[0, 1]))
            d["spearman_clock_vs_counts"] = {"min": min(rhos), "mean": float(np.mean(rhos))}
        out[kind] = d
    out["gpuclock_over_heuristic_true_E"] = (out["gpuclock"]["mean_E_true_work"]
                                             / out["heuristic"]["mean_E_true_work"])
    print(json.dumps(out))


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["default"]))
