"""Helpers shared by tests: scenario presets as plain dicts (oracle format)."""
from pathlib import Path

import yaml

from oracle import lbsim_oracle as O

PRESETS = Path(__file__).resolve().parent.parent / "paper_2104_11385_b200" / "scenarios"


def preset_doc(name):
    return yaml.safe_load((PRESETS / f"{name}.yaml").read_text())


def case_config(runs, name):
    """Oracle config for a fixture case in runs.json."""
    base = {"mini": "mini", "tight": "tight-memory", "default": "default"}
    ov = runs[name]["overrides"]
    if name in runs["_docs"]:
        cfg = O.config_from_doc(runs["_docs"][name])
    else:
        cfg = O.config_from_doc(preset_doc(base[name.split("_")[0]]))
    if "steps" in ov:
        cfg["steps"] = ov["steps"]
    if "policy" in ov:
        cfg = O.apply_policy(cfg, ov["policy"])
    if "cost" in ov:
        cfg["provider"] = ov["cost"]
    return cfg
