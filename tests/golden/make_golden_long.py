"""Long-run golden fixtures: the reference's own full `default` scenario
(2,000 steps, 801,499 particles, 24 ranks) run by the REAL reference
(lbsim, numpy kernels == compiled) in-process, for three policies
/ cost providers.  Stored compactly (sha256 of every per-step metric
column, the cost / count traces and the final state) in runs_long.json.

Run here (where /root/reference exists):  python tests/golden/make_golden_long.py
Nothing on the GPU box reads /root/reference; the GPU test is
tests/test_gpu_runs.py::test_long_run_matches_reference."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
from make_golden import OUT, advance, apply_overrides, init_scenario, load_spec, run_simulation, sha  # noqa: E402

CASES = {
    "default_full": {},                       # default.yaml as shipped (knapsack, heuristic)
    "default_full_measured": {"cost": "measured"},
    "default_full_sfc": {"policy": "sfc"},
}
COLUMNS = ("efficiency_before", "efficiency_after", "adopted", "compute_max", "comm_max",
           "gather", "redistribute", "walltime", "max_rank_particles", "oom")


def column_sha(metrics, name):
    v = [getattr(m, name) for m in metrics]
    dt = np.bool_ if name in ("adopted", "oom") else (
        np.int64 if name == "max_rank_particles" else np.float64)
    return sha(np.array(v, dtype=dt))


def main():
    out = {}
    for name, ov in CASES.items():
        spec = apply_overrides(load_spec("default"), **ov)
        res = run_simulation(spec.scenario, spec.policy, spec.build_provider())
        cfg = spec.scenario
        st = init_scenario(cfg)
        counts = []
        for _ in range(len(res.metrics)):
            st = advance(st, cfg)
            counts.append(st.per_box_particles.copy())
        out[name] = dict(
            overrides=ov,
            steps=len(res.metrics),
            metrics_sha={c: column_sha(res.metrics, c) for c in COLUMNS},
            cost_trace_sha=sha(res.cost_trace),
            count_trace_sha=sha(np.array(counts).astype(np.int64)),
            snapshots=[[int(s), o.tolist()] for s, o in res.adoption_snapshots],
            summary=res.summary,
            final_pos_sha=sha(st.positions),
            final_vel_sha=sha(st.velocities),
        )
        print(name, res.summary.get("adoption_count"), res.summary.get("mean_efficiency"), flush=True)
    (OUT / "runs_long.json").write_text(json.dumps(out, indent=0, sort_keys=True))


if __name__ == "__main__":
    main()
