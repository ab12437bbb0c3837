HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_kb128.so SHAPES=1x1 FLAGS=155,8347,8346,8344,8192 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | tail -5
