#!/bin/bash
timeout 300 python scripts/dbg_uq.py 2048 exact 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
SAN_TOOLS="memcheck" SAN_GROUPS="F X" timeout 900 bash scripts/gpu_sanitize.sh
