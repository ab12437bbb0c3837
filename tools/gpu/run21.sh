SHAPES=2x1 FLAGS=0,512 PRECS=fp32_tc timeout 300 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc" | tail -4
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --prec fp32_tc --no-cpu-baseline --no-e2e > gpurun_out/r21.json 2>gpurun_out/r21.err; python -c "import json; d=json.load(open('gpurun_out/r21.json')); print(d['ms_per_step'], d['value']/1e6, d['roofline']['kernel_ms'], d['roofline']['frac'], d['gpu_launches'])"
