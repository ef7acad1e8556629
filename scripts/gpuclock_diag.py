"""Diagnostics of the GpuClock tally at native size: per-box cycles per
particle (clk/count) spread and its dependence on the box's position."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2104_11385_b200 import scenarios as S  # noqa: E402
from paper_2104_11385_b200.workload import run_simulation  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 400
spec = S.apply_overrides(S.load_spec("default"), cost="gpuclock", steps=steps)
res = run_simulation(spec.scenario, spec.policy, spec.build_provider(), record_counts=True,
                     record_clock=True)
out = {}
for s in (0, 100, 149, 151, 200, steps - 1):
    if s >= steps:
        continue
    c = res.count_trace[s].astype(float)
    k = res.clock_trace[s].astype(float)
    big = c > 200
    r = k[big] / c[big]
    ids = np.nonzero(big)[0]
    out[s] = {"n_big": int(big.sum()), "ratio_mean": float(r.mean()),
              "ratio_cv": float(r.std() / r.mean()),
              "ratio_min": float(r.min()), "ratio_max": float(r.max()),
              "corr_ratio_boxid": float(np.corrcoef(r, ids)[0, 1]),
              "corr_ratio_count": float(np.corrcoef(r, c[big])[0, 1]),
              "ratio_by_row": {int(b // 30): round(float(np.mean(r[ids // 30 == b // 30])), 1)
                               for b in ids}}
print(json.dumps(out))
