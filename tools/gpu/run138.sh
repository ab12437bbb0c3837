timeout 600 python tools/tile_overhead.py 2>&1 | grep -v "^\[hdc"
for pr in fp32_tc bf16 tf32; do timeout 300 python bench.py --prec $pr --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$pr', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))"; done
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_train.py -q -x 2>&1 | tail -1
