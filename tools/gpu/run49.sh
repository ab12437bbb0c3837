timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "bf16 or tf32" 2>&1 | tail -2
SHAPES=2x1,1x1 FLAGS=0,155 PRECS=bf16,tf32,fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | tail -12
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_kb128.so SHAPES=2x1 FLAGS=0 PRECS=bf16,tf32 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | tail -2
