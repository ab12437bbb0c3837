timeout 1500 python -m pytest tests -q -m gpu -x -k "tc or train or fused" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"recheck|finalize" --csv --log-file gpurun_out/r114.csv python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu rc=$?
for c in cfg2 cfg4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done
