timeout 30 python tools/debug_encode.py bf16 33 7 17; echo rc=$?
timeout 30 python tools/debug_encode.py fp32_tc 33 7 17 noc; echo rc=$?
timeout 600 python -m pytest tests/test_gpu_train.py -x -q 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
