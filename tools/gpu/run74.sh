# CTA pair vs 2x1 cluster after CTA-scope expect_tx: timing, counters, timeline
SHAPES=2x1,2x1p FLAGS=0 PRECS=bf16,tf32 timeout 120 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | tail -6
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so SHAPES=2x1p FLAGS=4 PRECS=bf16 timeout 120 python tools/tc_timing.py 2>&1 | grep -v "rechecks" | sort | uniq -c | sort -rn | head -2
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so SHAPES=2x1p FLAGS=1024 PRECS=bf16 timeout 120 python tools/tc_timing.py 2>&1 | grep -A30 "timeline" | head -30
