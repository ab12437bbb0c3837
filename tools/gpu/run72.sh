# CTA-pair mode: watchdog diagnostics first (never hangs), then product build parity + timing
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so SHAPES=2x1p FLAGS=16384 PRECS=bf16 timeout 120 python tools/tc_timing.py 2>&1 | grep -v "rechecks" | head -40
export HDC_TC_CLUSTER=2x1p
timeout 200 python -m pytest tests/test_gpu_tc.py -x -q -k "bf16 or tf32" 2>&1 | tail -5
unset HDC_TC_CLUSTER
SHAPES=2x1,2x1p FLAGS=0 PRECS=bf16,tf32 timeout 120 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -6
