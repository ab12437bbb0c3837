mkdir -p gpurun_out/r117
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smallstream --launch-skip 2 --launch-count 1 -o gpurun_out/r117/full_smallstream_cfg3_n32 -f python bench.py --config cfg3_n32 --prec fp32 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r117/ncu.log 2>&1; echo "ncu rc=$?"
