timeout 600 python -m pytest tests -m gpu -x -q -k "host or abi or e2e" 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e6, d['e2e'], d['roofline']['traffic'])"
