SHAPES=1x1 FLAGS=155,2203 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | tail -2
SHAPES=1x1 FLAGS=3227 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -A 25 "timeline" | tail -24
