SHAPES=2x1 FLAGS=0,2,10,18,130,154,155,27 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | tail -8
SHAPES=2x1 FLAGS=6,158 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep "^\[hdc" | sort -u | tail -3
