"""Generate golden fixtures by running the REAL reference (lbsim) in-process.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The outputs are committed; nothing on the GPU box reads /root/reference.

Fixtures written (all small):
  kernels.npz     advance/bin inputs+outputs (reference test_kernels.py style)
  balancer.npz    random (cost, ranks) -> knapsack / sfc owners, efficiencies
  measured.npz    measured_cost noise vectors (PCG64 stream of cost.py:111)
  runs.json       whole-run results of scenario presets: metric columns,
                  sha256 of the cost trace / per-step counts, adoption
                  snapshots, summaries; per-step counts of early steps
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

os.environ["LBSIM_KERNELS"] = "python"   # numpy fallback == compiled, see SURVEY
sys.path.insert(0, "/root/reference/pkg/src")

import lbsim  # noqa: E402
from lbsim import _kernels_py  # noqa: E402
from lbsim.balancer import knapsack_assign, sfc_assign, efficiency_flagged  # noqa: E402
from lbsim.cost import CostVector, MeasurementConfig, measured_cost  # noqa: E402
from lbsim.decomposition import DistributionMapping, build_box_array, morton_order  # noqa: E402
from lbsim.scenarios import apply_overrides, load_spec, spec_from_dict  # noqa: E402
from lbsim.workload import advance, init_scenario, run_simulation  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def kernels_fixture():
    out = {}
    rng = np.random.default_rng(2024)
    for tag, n, extent, spill in (("a", 20000, 128.0, 0.1), ("b", 5000, 64.0, 0.02),
                                  ("c", 3, 8.0, 0.5), ("d", 4097, 96.0, 0.3)):
        pos = np.ascontiguousarray(rng.uniform(0, extent, size=(n, 2)))
        vel = np.ascontiguousarray(rng.normal(0, spill * extent, size=(n, 2)))
        p2, v2 = _kernels_py.advance_particles(pos, vel, extent, extent)
        out[f"{tag}_pos"], out[f"{tag}_vel"] = pos, vel
        out[f"{tag}_extent"] = np.array(extent)
        out[f"{tag}_out_pos"], out[f"{tag}_out_vel"] = p2, v2
        m = extent / 8
        out[f"{tag}_bins"] = _kernels_py.bin_particles(p2, m, 8, 8)
    # 25 chained steps (test_kernels.py:83-91 style)
    pos = np.ascontiguousarray(rng.uniform(0, 64.0, size=(5000, 2)))
    vel = np.ascontiguousarray(rng.normal(0, 0.02 * 64.0, size=(5000, 2)))
    out["chain_pos"], out["chain_vel"] = pos, vel
    for _ in range(25):
        pos, vel = _kernels_py.advance_particles(pos, vel, 64.0, 64.0)
    out["chain_out_pos"], out["chain_out_vel"] = pos, vel
    np.savez_compressed(OUT / "kernels.npz", **out)


def balancer_fixture():
    rng = np.random.default_rng(77)
    rows = []
    costs_all = []
    for i in range(400):
        nbz = int(rng.integers(1, 9))
        nbx = int(rng.integers(1, 9))
        n = nbz * nbx
        R = int(rng.integers(1, 10))
        kind = i % 4
        if kind == 0:      # integer costs: lots of ties
            c = rng.integers(0, 6, size=n).astype(float)
        elif kind == 1:    # heuristic-like (counts*0.75 + cells*0.25)
            c = 0.75 * rng.integers(0, 3000, size=n) + 0.25 * 256.0
        elif kind == 2:    # noisy measured-like
            c = (0.75 * rng.integers(0, 3000, size=n) + 64.0) * (1 + rng.uniform(-.05, .05, n))
        else:              # wide dynamic range
            c = rng.random(n) * 10.0 ** rng.uniform(-3, 4, n)
        cap = float(rng.choice([1.0, 1.25, 1.5, 2.0]))
        cv = CostVector(values=c)
        try:
            ks = knapsack_assign(cv, R, cap).owner
        except ValueError:
            ks = np.full(n, -1, dtype=np.int64)
        curve = morton_order(build_box_array((nbz, nbx), 1))
        sf = sfc_assign(cv, curve, R).owner
        e_ks = efficiency_flagged(cv, DistributionMapping(owner=ks, n_ranks=R))[0] if ks[0] >= 0 else -1.0
        e_sf = efficiency_flagged(cv, DistributionMapping(owner=sf, n_ranks=R))[0]
        rows.append((nbz, nbx, R, cap, e_ks, e_sf))
        costs_all.append((c, ks, sf, curve))
    out = {"meta": np.array(rows, dtype=float)}
    for i, (c, ks, sf, curve) in enumerate(costs_all):
        out[f"c{i}"], out[f"k{i}"], out[f"s{i}"], out[f"m{i}"] = c, ks, sf, curve
    # one large case: 900 boxes (default geometry), 8 and 24 ranks, noisy costs
    c = (0.75 * rng.integers(0, 60000, size=900) + 256.0) * (1 + rng.uniform(-.05, .05, 900))
    out["big_c"] = c
    for R in (8, 24):
        out[f"big_k{R}"] = knapsack_assign(CostVector(values=c), R).owner
        curve = morton_order(build_box_array((30, 30), 1))
        out[f"big_s{R}"] = sfc_assign(CostVector(values=c), curve, R).owner
    out["big_curve"] = morton_order(build_box_array((30, 30), 1))
    np.savez_compressed(OUT / "balancer.npz", **out)


def measured_fixture():
    out = {}
    for seed, step, n, amp in ((7, 0, 900, 0.05), (11, 123, 225, 0.05),
                               (13, 599, 900, 0.2), (0, 5, 17, 0.5),
                               (2 ** 40 + 3, 2 ** 33, 64, 0.05)):
        work = np.linspace(1.0, 1000.0, n)
        out[f"{seed}_{step}_{n}"] = measured_cost(
            work, MeasurementConfig(noise_amplitude=amp, seed=seed), step=step).values
    np.savez_compressed(OUT / "measured.npz", **out)


def scenario_docs():
    """YAML-equivalent documents for the extra configs."""
    c1 = dict(scenario_id="c1-uniform", domain=dict(extent=[128, 128], box_size=32),
              ranks=8, blob=dict(center=[64.0, 64.0], core_radius=91.0, edge_scale=0.0,
                                 particles_per_cell=8.0),
              kick=dict(step=0, speed=0.0), steps=40, seed=1,
              balance=dict(strategy="knapsack", interval=10, threshold=0.10))
    small = dict(scenario_id="small", domain=dict(extent=[96, 96], box_size=16), ranks=4,
                 blob=dict(center=[48.0, 48.0], core_radius=16.0, edge_scale=2.0,
                           particles_per_cell=6.0),
                 kick=dict(step=3, speed=0.4, drift=0.1), steps=40, seed=21)
    leaky = dict(scenario_id="leaky", domain=dict(extent=[64, 64], box_size=8), ranks=3,
                 blob=dict(center=[20.0, 40.0], core_radius=10.0, edge_scale=3.0,
                           particles_per_cell=3.5),
                 kick=dict(step=2, speed=1.7, drift=0.6), steps=30, seed=5,
                 balance=dict(strategy="sfc", interval=3, threshold=0.0))
    return {"c1": c1, "small": small, "leaky": leaky}


def run_fixture():
    cases = {
        "mini": (load_spec("mini"), {}),
        "mini_none": (load_spec("mini"), {"policy": "none"}),
        "mini_static": (load_spec("mini"), {"policy": "static"}),
        "mini_sfc": (load_spec("mini"), {"policy": "sfc"}),
        "mini_measured": (load_spec("mini"), {"cost": "measured"}),
        "mini_instrumented": (load_spec("mini"), {"cost": "instrumented", "steps": 60}),
        "tight": (load_spec("tight-memory"), {}),
        "tight_none": (load_spec("tight-memory"), {"policy": "none"}),
        "default_short": (load_spec("default"), {"steps": 170, "cost": "measured"}),
    }
    for name, doc in scenario_docs().items():
        cases[name] = (spec_from_dict(doc), {})
    out = {}
    for name, (spec, ov) in cases.items():
        spec = apply_overrides(spec, **ov)
        res = run_simulation(spec.scenario, spec.policy, spec.build_provider())
        cfg = spec.scenario
        # per-step counts by re-stepping the state (same kernels as the run)
        st = init_scenario(cfg)
        counts = []
        for _ in range(len(res.metrics)):
            st = advance(st, cfg)
            counts.append(st.per_box_particles.copy())
        counts = np.array(counts)
        ms = res.metrics
        out[name] = dict(
            overrides=ov,
            doc=None,
            metrics={
                "eff_before": [m.efficiency_before for m in ms],
                "eff_after": [m.efficiency_after for m in ms],
                "adopted": [bool(m.adopted) for m in ms],
                "compute_max": [m.compute_max for m in ms],
                "comm_max": [m.comm_max for m in ms],
                "gather": [m.gather for m in ms],
                "redistribute": [m.redistribute for m in ms],
                "walltime": [m.walltime for m in ms],
                "max_rank_particles": [m.max_rank_particles for m in ms],
                "oom": [bool(m.oom) for m in ms],
            },
            cost_trace_sha=sha(res.cost_trace),
            cost_trace_head=res.cost_trace[:3].tolist(),
            count_trace_sha=sha(counts.astype(np.int64)),
            counts_first=counts[0].tolist(),
            counts_last=counts[-1].tolist(),
            initial_owner=res.initial_owner.tolist(),
            snapshots=[[int(s), o.tolist()] for s, o in res.adoption_snapshots],
            summary=res.summary,
            final_pos_sha=sha(st.positions),
            final_vel_sha=sha(st.velocities),
            init_pos_sha=sha(init_scenario(cfg).positions),
            n_init=int(init_scenario(cfg).n_particles),
        )
    out["_docs"] = scenario_docs()
    (OUT / "runs.json").write_text(json.dumps(out, indent=0, sort_keys=True))


if __name__ == "__main__" and not any(a.startswith("--cli") for a in sys.argv):
    print("reference lbsim", lbsim.__version__, "backend", lbsim.KERNEL_BACKEND)
    kernels_fixture()
    balancer_fixture()
    measured_fixture()
    run_fixture()
    cli_fixture()
    for p in sorted(OUT.iterdir()):
        print(p.name, p.stat().st_size)


def cli_fixture():
    """sha256 of the reference CLI's own output files (lbsim/cli.py:65-101)."""
    import tempfile

    from lbsim import cli
    cases = {"mini": ["--scenario", "mini"],
             "mini_sfc": ["--scenario", "mini", "--policy", "sfc"],
             "mini_measured": ["--scenario", "mini", "--cost", "measured", "--steps", "120"],
             "tight_none": ["--scenario", "tight-memory", "--policy", "none"],
             "tight": ["--scenario", "tight-memory", "--steps", "200"]}
    out = {}
    for name, argv in cases.items():
        with tempfile.TemporaryDirectory() as d:
            rc = cli.main(["run", *argv, "--out", d])
            out[name] = {"argv": argv, "rc": rc,
                         **{f: hashlib.sha256((Path(d) / f).read_bytes()).hexdigest()
                            for f in ("metrics.csv", "cost_trace.csv", "mappings.csv",
                                      "summary.json")}}
            rd = Path(d) / "replay"
            cli.main(["replay", "--run-dir", d, "--out", str(rd)])
            out[name]["replay_metrics.csv"] = hashlib.sha256(
                (rd / "replay_metrics.csv").read_bytes()).hexdigest()
    (OUT / "cli.json").write_text(json.dumps(out, indent=1, sort_keys=True))


FIT_POINTS = [(1, 812.5), (2, 431.0), (4, 239.25), (8, 137.75), (16, 84.0)]
COMPARE_RUNS = {"dyn": ["--scenario", "mini", "--steps", "150"],
                "sfc": ["--scenario", "mini", "--steps", "150", "--policy", "sfc"],
                "none": ["--scenario", "mini", "--steps", "150", "--policy", "none"]}


def cli_tools_fixture():
    """Stdout of the reference CLI's `fit` and `compare` (lbsim/cli.py:328-371)
    on fixed inputs: a nodes,walltime CSV and three mini runs."""
    import contextlib
    import io
    import tempfile

    from lbsim import cli
    out = {"fit_points": FIT_POINTS, "compare_runs": list(COMPARE_RUNS.items())}
    with tempfile.TemporaryDirectory() as d:
        pts = Path(d) / "points.csv"
        pts.write_text("nodes,walltime\n" + "".join(f"{n},{w}\n" for n, w in FIT_POINTS))
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = cli.main(["fit", "--points", str(pts), "--e0", "0.3155", "--e0", "0.2"])
        out["fit"] = {"rc": rc, "stdout": buf.getvalue()}
        dirs = []
        for name, argv in COMPARE_RUNS.items():
            rd = Path(d) / name
            cli.main(["run", *argv, "--out", str(rd)])
            dirs.append(str(rd))
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = cli.main(["compare", *dirs])
        out["compare"] = {"rc": rc, "stdout": buf.getvalue()}
    (OUT / "cli_tools.json").write_text(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__" and "--cli" in sys.argv:
    cli_fixture()

if __name__ == "__main__" and "--cli-tools" in sys.argv:
    cli_tools_fixture()
