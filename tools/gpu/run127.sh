mkdir -p gpurun_out/r127
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ffma --launch-skip 1 --launch-count 1 -o gpurun_out/r127/full_ffma_cfg2 -f python bench.py --config cfg2 --prec fp32 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r127/ncu.log 2>&1; echo "ncu rc=$?"
