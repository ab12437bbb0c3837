BENCH_LIKE=1 timeout 200 python tools/e2e_probe.py 2>&1 | tail -1
BENCH_LIKE=1 PREC=bf16 timeout 200 python tools/e2e_probe.py 2>&1 | tail -1
for pr in fp32_tc bf16; do timeout 300 python bench.py --prec $pr --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$pr', round(d['e2e']['value']/1e6,2), 'M/s e2e')"; done
timeout 600 python -m pytest tests/test_gpu_small.py -q -x 2>&1 | tail -1
