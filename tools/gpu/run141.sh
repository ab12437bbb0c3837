FS=128,640 PRECS=fp32_tc timeout 300 python tools/tile_overhead.py 2>&1 | grep "kernel"
for c in cfg2 cfg4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_train.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -1
