for i in 1 2; do BENCH_LIKE=1 timeout 200 python tools/e2e_probe.py 2>&1 | tail -1; BENCH_LIKE=1 PREC=bf16 timeout 200 python tools/e2e_probe.py 2>&1 | tail -1; done
timeout 120 python tools/h2d_bw.py 2>&1 | head -3
for pr in fp32_tc bf16; do timeout 300 python bench.py --prec $pr --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$pr', d['e2e'])"; done
