timeout 600 python -m pytest tests/test_gpu_sharding.py tests/test_gpu_small.py -x -q 2>&1 | tail -4
