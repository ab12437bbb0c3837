timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for c in cfg2 cfg4 cfg5; do for pr in fp32_tc bf16; do timeout 600 python bench.py --config $c --prec $pr --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$pr', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done; done
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"limb_rows|round_rows" --csv --log-file gpurun_out/r112.csv python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu rc=$?
