python -m pytest tests/test_gpu_pic.py -x -q 2>&1 | tail -25
