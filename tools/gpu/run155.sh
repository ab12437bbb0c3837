for c in cfg4 cfg5 cfg2; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))"; done
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -k "fp32_tc" 2>&1 | tail -1
