for n in 2048 16384; do
NROWS=$n HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so FLAGS=0,4 PRECS=bf16 timeout 120 python tools/tc_timing.py 2>&1 | grep -v "rechecks" | sort | uniq -c | sort -rn | head -3
done
NROWS=2048 HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so FLAGS=1024 PRECS=bf16 timeout 120 python tools/tc_timing.py 2>&1 | grep -A70 "timeline" | head -72
