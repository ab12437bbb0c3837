mkdir -p gpurun_out
for sh in 1x2 2x2 1x4; do
  HDC_TC_CLUSTER=$sh timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "cfg2" 2>&1 | tail -2 | sed "s/^/$sh: /"
done
for pr in bf16 fp32_tc; do
  PRECS=$pr SHAPES=1x1 FLAGS=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_tc --launch-skip 3 --launch-count 1 -o gpurun_out/r6_$pr -f python tools/tc_timing.py > gpurun_out/r6_ncu_$pr.log 2>&1
  tail -3 gpurun_out/r6_ncu_$pr.log
done
