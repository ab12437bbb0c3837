SHAPES=1x1,2x1 FLAGS=0,26 PRECS=bf16,fp32_tc,tf32 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -12
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
