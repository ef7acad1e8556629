#!/bin/bash
for v in buggy ""; do
LBX_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_pic_fast.py -q -x -k "large_sparse" 2>&1 | grep -E "Error|passed|failed" | head -3
done
