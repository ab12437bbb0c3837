SHAPES=2x1,1x1 FLAGS=4 PRECS=fp32_tc,bf16 timeout 300 python tools/tc_timing.py 2>&1 | grep -v "rechecks" | awk '/tc debug/{l=$0} !/tc debug/{print; if (l) print l}' | tail -8
