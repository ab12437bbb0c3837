BENCH_LIKE=1 timeout 200 python tools/e2e_probe.py
BENCH_LIKE=1 PREC=bf16 timeout 200 python tools/e2e_probe.py
