for i in 1 2; do
SHAPES=2x1 FLAGS=0 PRECS=fp32_tc,bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | sed "s|^|new |" | tail -2
SHAPES=2x1 FLAGS=0 PRECS=fp32_tc,bf16 timeout 300 python exp/old/tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | sed "s|^|old |" | tail -2
done
