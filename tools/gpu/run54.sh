for L in paper_2506_09282_b200/lib/libhdc.so exp/libhdc_3af93a6.so paper_2506_09282_b200/lib/libhdc.so exp/libhdc_3af93a6.so; do
HDC_LIB_PATH=$L SHAPES=2x1 FLAGS=0 PRECS=fp32_tc,bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | sed "s|^|$L |" | tail -2
done
