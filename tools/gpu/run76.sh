timeout 200 python tools/e2e_probe.py
PREC=bf16 timeout 200 python tools/e2e_probe.py
