#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_pic_fast.py -q -x -k "large_sparse" 2>&1 | tail -3
