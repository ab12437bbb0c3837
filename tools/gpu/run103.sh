timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_train.py tests/test_gpu_fused.py -x -q 2>&1 | tail -2
timeout 300 python tools/smalln_probe.py 2>&1 | grep -v "^\[hdc"
