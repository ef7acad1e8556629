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
