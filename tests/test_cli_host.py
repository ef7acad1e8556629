"""CLI writers and replay on CPU: the oracle's whole-run results written by
our writers must hash to the reference CLI's own files, and replay (our C++
balancer) must reproduce the reference's replay output."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import lbsim_oracle as O
from tests.scenario_util import preset_doc

G = Path(__file__).resolve().parent / "golden"


def sha_file(p):
    return hashlib.sha256(Path(p).read_bytes()).hexdigest()


def result_from_oracle(cfg, name):
    from paper_2104_11385_b200.workload import RunResult, StepMetrics
    r = O.run_simulation(cfg)
    m = r["metrics"]
    metrics = [StepMetrics(int(m["step"][i]), float(m["eff_before"][i]), float(m["eff_after"][i]),
                           bool(m["adopted"][i]), float(m["compute_max"][i]),
                           float(m["comm_max"][i]), float(m["gather"][i]),
                           float(m["redistribute"][i]), float(m["walltime"][i]),
                           int(m["max_rank_particles"][i]), bool(m["oom"][i]))
               for i in range(len(m["step"]))]
    nbz, nbx = cfg["extent"][0] // cfg["box_size"], cfg["extent"][1] // cfg["box_size"]
    pk = {"heuristic": "heuristic", "measured": "measured", "instrumented": "instrumented"}
    s = r["summary"]
    total = cfg["steps"]
    summary = {"scenario_id": cfg["scenario_id"], "n_ranks": cfg["ranks"],
               "n_boxes": nbz * nbx, "box_grid": [nbz, nbx], "seed": cfg["seed"],
               "policy": ("dynamic" if cfg["interval"] <= total else
                          "static" if cfg["static_step"] is not None else "none"),
               "strategy": cfg["strategy"], "interval": cfg["interval"],
               "improvement_threshold": cfg["threshold"],
               "threshold_mode": cfg["threshold_mode"], "static_step": cfg["static_step"],
               "provider": pk[cfg["provider"]],
               "overhead_factor": (cfg["instrumented_overhead"]
                                   if cfg["provider"] == "instrumented" else 1.0),
               "total_steps": total, **{k: s[k] for k in (
                   "completed_steps", "completion_fraction", "total_walltime",
                   "mean_efficiency", "adoption_count", "attempt_count", "oom",
                   "final_particles")}}
    return RunResult(metrics=metrics, summary=summary, cost_trace=r["cost_trace"],
                     initial_owner=r["initial_owner"], adoption_snapshots=r["snapshots"])


CASES = {"mini": ("mini", {}), "mini_sfc": ("mini", {"policy": "sfc"}),
         "mini_measured": ("mini", {"cost": "measured", "steps": 120}),
         "tight_none": ("tight-memory", {"policy": "none"})}


@pytest.mark.parametrize("name", list(CASES))
def test_writers_and_replay_byte_identical(tmp_path, name):
    from paper_2104_11385_b200 import cli
    want = json.loads((G / "cli.json").read_text())[name]
    base, kw = CASES[name]
    cfg = O.config_from_doc(preset_doc(base))
    if "steps" in kw:
        cfg["steps"] = kw["steps"]
    if "policy" in kw:
        cfg = O.apply_policy(cfg, kw["policy"])
    if "cost" in kw:
        cfg["provider"] = kw["cost"]
    cli.write_run_outputs(tmp_path, result_from_oracle(cfg, name))
    for f in ("metrics.csv", "cost_trace.csv", "mappings.csv", "summary.json"):
        assert sha_file(tmp_path / f) == want[f], (name, f)
    assert cli.main(["replay", "--run-dir", str(tmp_path), "--out", str(tmp_path / "r")]) == 0
    assert sha_file(tmp_path / "r" / "replay_metrics.csv") == want["replay_metrics.csv"]


def test_cli_usage_errors(tmp_path):
    from paper_2104_11385_b200 import cli
    assert cli.main(["run", "--scenario", "nope", "--out", str(tmp_path)]) == 1
    assert cli.main(["replay"]) == 1
    assert cli.main(["bogus"]) == 1


def test_fit_and_compare_match_reference_stdout(tmp_path, capsys):
    """`fit` and `compare` (cli.py:328-371) print exactly what the reference
    CLI printed on the same inputs (tests/golden/cli_tools.json); the run
    directories come from our writers over oracle runs (byte-identical to the
    reference's, test above)."""
    from paper_2104_11385_b200 import cli
    want = json.loads((G / "cli_tools.json").read_text())
    pts = tmp_path / "points.csv"
    pts.write_text("nodes,walltime\n" + "".join(f"{n},{w}\n" for n, w in want["fit_points"]))
    capsys.readouterr()
    assert cli.main(["fit", "--points", str(pts), "--e0", "0.3155", "--e0", "0.2"]) == 0
    assert capsys.readouterr().out == want["fit"]["stdout"]
    dirs = []
    for name, argv in want["compare_runs"]:      # in the reference's order
        cfg = O.config_from_doc(preset_doc("mini"))
        cfg["steps"] = int(argv[argv.index("--steps") + 1])
        if "--policy" in argv:
            cfg = O.apply_policy(cfg, argv[argv.index("--policy") + 1])
        d = tmp_path / name
        cli.write_run_outputs(d, result_from_oracle(cfg, name))
        dirs.append(str(d))
    capsys.readouterr()
    assert cli.main(["compare", *dirs]) == 0
    assert capsys.readouterr().out == want["compare"]["stdout"]
    assert cli.main(["compare", dirs[0]]) == 1          # needs two runs (usage error)
