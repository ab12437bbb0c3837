mkdir -p gpurun_out
BENCH_LIKE=1 HDC_HOST_TRACE=1 timeout 200 python tools/e2e_probe.py > gpurun_out/r90.log 2>&1
