timeout 200 python tools/e2e_probe.py
PREC=bf16 timeout 200 python tools/e2e_probe.py
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fused.py -x -q 2>&1 | tail -3
