timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_train.py -x -q 2>&1 | tail -2
for v in 0 1; do if [ $v = 1 ]; then export HDC_NO_PDL=1; fi
for pr in fp32_tc bf16; do timeout 300 python bench.py --prec $pr --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nopdl=$v', '$pr', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done; done
