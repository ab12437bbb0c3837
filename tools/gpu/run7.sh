SHAPES=1x1 FLAGS=0,2,8,10,18,26,24,16 PRECS=bf16 timeout 300 python tools/tc_timing.py 2>&1 | tail -12
cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_microbench mma_microbench.cu && ./mma_microbench
