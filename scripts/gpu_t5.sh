#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x -k "pic" 2>&1 | tail -15
