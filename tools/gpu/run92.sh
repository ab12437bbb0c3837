FLAGS=0 PRECS=fp32_tc timeout 120 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc"
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_kb8.so FLAGS=0 PRECS=fp32_tc timeout 120 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc"
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_kb8.so timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "fp32_tc and cfg2" 2>&1 | tail -2
