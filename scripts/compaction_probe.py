#!/usr/bin/env python
"""Leaver-heavy step (bench.py compaction_leavers workload) for ncu: 100 M
particles uniform over 960^2, v ~ N(0, 2), random order; prints the bench
line's compaction numbers (step - push kernel) for comparison."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
print(json.dumps(bench.compaction_leavers(torch.device("cuda:0"), steps=steps)))
