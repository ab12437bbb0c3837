SHAPES=2x1 FLAGS=0,2,8,16,24,18,4 PRECS=fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -7
SHAPES=2x1 FLAGS=4 PRECS=fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep "^\[hdc" | tail -1
