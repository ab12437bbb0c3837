SHAPES=2x1,2x1p FLAGS=0 PRECS=bf16,tf32 timeout 120 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks"
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_nat2.so SHAPES=2x1,2x1p FLAGS=0 PRECS=bf16,tf32 timeout 120 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | sed 's/^/nat2 /'
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_nat2.so timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "bf16 or tf32" 2>&1 | tail -2
