SHAPES=1x1 FLAGS=1179 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -A 66 "timeline" | tail -66
