timeout 120 python tools/h2d_bw.py 2>&1 | head -4
BENCH_LIKE=1 timeout 200 python tools/e2e_probe.py 2>&1 | tail -1
timeout 120 python tools/h2d_bw.py 2>&1 | head -2
nproc; cat /proc/loadavg; free -g | head -2
