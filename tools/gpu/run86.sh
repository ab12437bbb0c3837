timeout 300 python -m pytest tests/test_gpu_small.py -x -q 2>&1 | tail -3
timeout 200 python tools/e2e_probe.py 2>&1 | grep infer_host
PREC=bf16 timeout 200 python tools/e2e_probe.py 2>&1 | grep infer_host
timeout 300 python bench.py --steps 20 --warmup 5 2>&1 | tail -1
