for c in cfg5 cfg4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r69_$c.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r69_$c.json')); r=d['roofline']; print('$c', round(d['ms_per_step'],3), round(r['kernel_ms'],3), round(d['value']/1e6,3), round(r['frac'],3))"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | grep gpu__time > gpurun_out/r69_launch.csv; python - <<'PY'
import csv
for r in csv.reader(open("gpurun_out/r69_launch.csv")):
    print(r[4][:60], r[-1])
PY
