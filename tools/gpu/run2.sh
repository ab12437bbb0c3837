# K4 tile-width / Stage II A/B (invoked through gpurun)
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 120 $B --prec bf16 > gpurun_out/r2_bf16.json 2> gpurun_out/r2_bf16.err
timeout 120 $B --prec fp32_tc > gpurun_out/r2_i8.json 2> gpurun_out/r2_i8.err
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_s2f.so timeout 120 $B --prec fp32_tc > gpurun_out/r2_i8_s2f.json 2> gpurun_out/r2_i8_s2f.err
timeout 120 $B --prec tf32 > gpurun_out/r2_tf32.json 2> gpurun_out/r2_tf32.err
for p in fp32_tc bf16; do HDC_TC_DEBUG=4 timeout 120 python bench.py --steps 1 --warmup 2 --prec $p --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/r2_dbg_$p.err; done
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -15 > gpurun_out/r2_pytest_tc.log
cat gpurun_out/r2_pytest_tc.log
for f in gpurun_out/r2_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['ms_per_step'], d['value']/1e6, d['roofline']['kernel_ms'], d['roofline']['frac'])"; done
grep -h "tc debug" gpurun_out/r2_dbg*.err | tail -2; tail -3 gpurun_out/r2_*.err
