for s in 20 100; do timeout 300 python bench.py --steps $s --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['steps'], d['value'], d['e2e'])"; done
timeout 300 python bench.py --steps 20 --warmup 5 --prec bf16 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['steps'], d['value'], d['e2e'])"
