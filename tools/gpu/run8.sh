SHAPES=1x1 FLAGS=26,30,4 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | tail -12
