SHAPES=2x1,1x1 FLAGS=0,529,25,2 PRECS=fp32_tc,bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | tail -16
