SHAPES=1x1 FLAGS=0,26 PRECS=bf16,fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -4
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_e4.so SHAPES=1x1 FLAGS=0,26 PRECS=bf16,fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -4
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "edge_grid and (bf16 or fp32_tc)" 2>&1 | tail -2
