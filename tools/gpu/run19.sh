SHAPES=2x1 FLAGS=0,512,528 PRECS=fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -4
