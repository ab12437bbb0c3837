SHAPES=2x1 FLAGS=0 PRECS=bf16,tf32,fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | tail -3
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so SHAPES=2x1 FLAGS=0,8346,8347 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | tail -3
