timeout 30 python tools/debug_encode.py bf16 33 7 17; echo rc=$?
timeout 30 python tools/debug_encode.py fp32_tc 33 7 17; echo rc=$?
HDC_TC_CLUSTER=1x1 timeout 30 python tools/debug_encode.py fp32_tc 33 7 17; echo rc=$?
timeout 30 python tools/debug_encode.py fp32_tc 33 7 17 noc; echo rc=$?
