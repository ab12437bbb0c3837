timeout 600 python -m pytest tests/test_gpu_train.py tests/test_gpu_tc.py -x -q -k "fp32_tc or encode or bundle or train or cancel" 2>&1 | tail -2
for i in 1 2; do
SHAPES=2x1 FLAGS=0 PRECS=fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | sed "s|^|new |" | tail -1
SHAPES=2x1 FLAGS=0 PRECS=fp32_tc timeout 300 python exp/old/tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | sed "s|^|old |" | tail -1
done
