FLAGS=0 PRECS=fp32_tc timeout 120 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc"
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
