# K4 rework: early accumulator release, opportunistic Stage II, H in TMEM (invoked through gpurun)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "edge_grid and (bf16 or fp32_tc)" 2>&1 | tail -25 > gpurun_out/r3_pytest_a.log
cat gpurun_out/r3_pytest_a.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for p in bf16 fp32_tc tf32; do timeout 120 $B --prec $p > gpurun_out/r3_$p.json 2> gpurun_out/r3_$p.err; done
for p in fp32_tc bf16; do HDC_TC_DEBUG=4 timeout 120 python bench.py --steps 1 --warmup 2 --prec $p --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/r3_dbg_$p.err; done
for f in gpurun_out/r3_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['ms_per_step'], d['value']/1e6, d['roofline']['kernel_ms'], d['roofline']['frac'])"; done
grep -h "tc debug" gpurun_out/r3_dbg*.err | tail -2
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -15 > gpurun_out/r3_pytest_tc.log
cat gpurun_out/r3_pytest_tc.log
