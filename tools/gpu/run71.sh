# CTA-pair (cta_group::2) mode: parity under HDC_TC_CLUSTER=2x1p, then timing vs the 2x1 cluster
export HDC_TC_CLUSTER=2x1p
timeout 240 python -m pytest tests/test_gpu_tc.py -x -q -k "bf16 or tf32" 2>&1 | tail -5
unset HDC_TC_CLUSTER
SHAPES=2x1,2x1p FLAGS=0 PRECS=bf16,tf32 timeout 200 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -6
