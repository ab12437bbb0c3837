for L in libhdc libhdc_spin libhdc_hint; do
echo $L
HDC_LIB_PATH=paper_2506_09282_b200/lib/$L.so SHAPES=1x1 FLAGS=0,27 PRECS=bf16,fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -4
done
