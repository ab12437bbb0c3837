for v in old mid; do
SHAPES=2x1 FLAGS=0 PRECS=fp32_tc timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fused_tc --csv python exp/$v/tools/tc_timing.py 2>/dev/null | grep gpu__time | awk -F'","' -v v=$v '{print v, $NF}' | tail -2
done
SHAPES=2x1 FLAGS=0 PRECS=fp32_tc timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fused_tc --csv python tools/tc_timing.py 2>/dev/null | grep gpu__time | awk -F'","' '{print "new", $NF}' | tail -2
