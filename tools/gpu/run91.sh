for n in 2048 8192 16384; do
NROWS=$n HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so SHAPES=1x1 FLAGS=0,8346,8347 PRECS=bf16 timeout 200 python tools/tc_timing.py 2>&1 | grep -v "rechecks\|^\[hdc" | sed "s/^/n=$n /"
done
