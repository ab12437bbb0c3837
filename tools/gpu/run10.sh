SHAPES=1x1 FLAGS=26,154,282,410 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -12
