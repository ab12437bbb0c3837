CFG=cfg4 FLAGS=0 PRECS=fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc"
CFG=cfg5 FLAGS=0 PRECS=fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc"
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"recheck|finalize" --csv --log-file gpurun_out/r113.csv python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu rc=$?
