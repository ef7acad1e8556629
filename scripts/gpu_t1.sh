#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_pic.py -q -x -k "round_trip" 2>&1 | tail -30
