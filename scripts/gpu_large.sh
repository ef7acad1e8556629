#!/bin/bash
timeout 900 python scripts/dbg_large.py 2>&1 | grep -vE "^\s+File|^\s+\^" | tail -20
