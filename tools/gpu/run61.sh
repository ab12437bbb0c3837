SHAPES=2x1 FLAGS=0 PRECS=fp32_tc,bf16 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fused_tc --csv python tools/tc_timing.py 2>/dev/null | grep gpu__time > gpurun_out/r61.csv; python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r61.csv")))
for r in rows:
    print(r[4][:40], r[-1])
PY
