for L in libhdc libhdc_cw9 libhdc_cw10; do
for c in cfg3_n1 cfg3_n4 cfg3_n16 cfg3_n32; do HDC_LIB_PATH=paper_2506_09282_b200/lib/$L.so timeout 300 python bench.py --config $c --prec fp32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', '$c', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['kernel_ms']*1000,1))"; done; done
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_cw10.so timeout 600 python -m pytest tests/test_gpu_small.py tests/test_gpu_sharding.py -q -x 2>&1 | tail -1
HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_cw9.so timeout 600 python -m pytest tests/test_gpu_small.py tests/test_gpu_sharding.py -q -x 2>&1 | tail -1
