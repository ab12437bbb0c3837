# validation + baseline numbers (invoked through gpurun)
mkdir -p gpurun_out
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for p in fp32_tc bf16 tf32; do timeout 300 python bench.py --steps 10 --warmup 3 --prec $p --no-cpu-baseline --no-e2e > gpurun_out/b_cfg2_$p.json 2> gpurun_out/b_cfg2_$p.err; done
for p in fp32_tc bf16; do HDC_TC_DEBUG=4 timeout 300 python bench.py --steps 1 --warmup 3 --prec $p --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/dbg_cfg2_$p.err; done
timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --prec fp32 --no-cpu-baseline --no-e2e > gpurun_out/b_cfg3.json 2> gpurun_out/b_cfg3.err
timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --prec bf16 --no-cpu-baseline --no-e2e > gpurun_out/b_cfg4_bf16.json 2> gpurun_out/b_cfg4.err
cat gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/b_*.json; grep "tc debug" gpurun_out/dbg*.err | tail -4
