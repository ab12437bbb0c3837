mkdir -p gpurun_out
timeout 300 python tools/tc_timing.py 2>&1 | tail -30 | tee gpurun_out/r4_timing.log
