"""Dump GpuClock traces at the reference's C2 size for offline analysis."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2104_11385_b200 import scenarios as S  # noqa: E402
from paper_2104_11385_b200.workload import run_simulation  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 400
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/gpuclock_traces.npz"
spec = S.apply_overrides(S.load_spec("default"), cost="gpuclock", steps=steps)
res = run_simulation(spec.scenario, spec.policy, spec.build_provider(), record_counts=True,
                     record_clock=True)
np.savez_compressed(out, clock=res.clock_trace, counts=res.count_trace, cost=res.cost_trace)
