for i in 1 2; do
SHAPES=2x1 FLAGS=0 PRECS=fp32_tc,bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | sed "s|^|prod |" | tail -2
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so SHAPES=2x1 FLAGS=0 PRECS=fp32_tc,bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | sed "s|^|diag |" | tail -2
done
