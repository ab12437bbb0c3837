SHAPES=2x1,2x1p FLAGS=0 PRECS=bf16,tf32 timeout 200 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks"
CFG=cfg4 SHAPES=2x1,2x1p FLAGS=0 PRECS=bf16 timeout 200 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks"
