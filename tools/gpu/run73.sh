# CTA pair vs 2x1 cluster: per-role wait counters and CTA-0 stage timeline (diagnostics build)
for S in 2x1 2x1p; do
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so SHAPES=$S FLAGS=0,4 PRECS=bf16 timeout 120 python tools/tc_timing.py 2>&1 | grep -v "rechecks" | sort | uniq -c | sort -rn | head -4
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so SHAPES=$S FLAGS=1024 PRECS=bf16 timeout 120 python tools/tc_timing.py 2>&1 | grep -A40 "timeline" | head -42
done
