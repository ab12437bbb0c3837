for n in 2048 16384; do
NROWS=$n HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so FLAGS=1024 PRECS=fp32_tc timeout 120 python tools/tc_timing.py 2>&1 | grep -A42 "timeline" | head -42
done
