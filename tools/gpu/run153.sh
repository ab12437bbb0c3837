timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -1
timeout 600 python bench.py --config cfg1 --prec fp32 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1 fp32', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
