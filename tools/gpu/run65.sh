HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so SHAPES=1x1 FLAGS=8347,155,8346 PRECS=bf16 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:fused_tc --csv python tools/tc_timing.py 2>/dev/null | grep "gpu__time\|cycles_elapsed" > gpurun_out/r65.csv; python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r65.csv")))
for r in rows:
    print(r[-3], r[-1])
PY
