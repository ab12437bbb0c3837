SHAPES=1x1 FLAGS=0,30,26 PRECS=bf16,fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -12
