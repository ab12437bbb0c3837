SHAPES=2x1 FLAGS=0,512 PRECS=fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -4
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "fp32_tc or cancel or ffma" 2>&1 | tail -2
