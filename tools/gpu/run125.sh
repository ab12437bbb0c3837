for c in cfg4 cfg5 cfg2; do CFG=$c SHAPES=2x1,2x1p FLAGS=0 PRECS=tf32 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks"; done
