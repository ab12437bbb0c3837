mkdir -p gpurun_out
for sh in 1x2 2x1 2x2 1x4 1x1; do
  HDC_TC_CLUSTER=$sh timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "edge_grid or cfg2" 2>&1 | tail -3 | sed "s/^/$sh: /"
done
SHAPES=1x1,1x2,2x1,2x2,1x4 FLAGS=0,16 PRECS=fp32_tc,bf16,tf32 timeout 300 python tools/tc_timing.py 2>&1 | tail -40
