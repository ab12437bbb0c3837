timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_train.py -x -q -k "fp32_tc or encode or bundle or train" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"limb_rows|round_rows|recheck|finalize" --csv --log-file gpurun_out/r105.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu rc=$?
