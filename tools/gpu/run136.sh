mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r136.csv python bench.py --config cfg4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu rc=$?
