SHAPES=1x1 FLAGS=155,4251,0,4096 PRECS=bf16,fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | tail -8
SHAPES=1x1 FLAGS=5275 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -A 25 "timeline" | tail -14
