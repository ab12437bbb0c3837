HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so SHAPES=1x1,2x1 FLAGS=0,32768,8194,40962,8346 PRECS=bf16 timeout 200 python tools/tc_timing.py 2>&1 | grep -v "rechecks\|^\[hdc"
