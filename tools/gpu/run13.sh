SHAPES=1x1 FLAGS=27,26,25,31 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -5
SHAPES=1x1 FLAGS=31 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep "^\[hdc" | tail -1
