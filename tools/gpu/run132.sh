for i in 1 2; do
for pr in fp32_tc bf16; do
(cd exp/old && timeout 300 python bench.py --prec $pr --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', '$pr', round(d['e2e']['value']/1e6,2), 'M/s', round(d['ms_per_step'],4))")
timeout 300 python bench.py --prec $pr --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', '$pr', round(d['e2e']['value']/1e6,2), 'M/s', round(d['ms_per_step'],4))"
done; done
