timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "fp32_tc or cancel" 2>&1 | tail -1
for L in paper_2506_09282_b200/lib/libhdc.so paper_2506_09282_b200/lib/libhdc_u5.so; do
HDC_LIB_PATH=$L SHAPES=2x1 FLAGS=0 PRECS=fp32_tc,bf16 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fused_tc --csv python tools/tc_timing.py 2>/dev/null | grep gpu__time > gpurun_out/r63.csv; python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r63.csv")))
for r in rows[-2:] + rows[8:9]:
    print(r[4][:45], r[-1])
PY
done
