for c in cfg3_n1 cfg3_n32; do HDC_SMALL_DEBUG=1 timeout 300 python bench.py --config $c --steps 3 --warmup 2 --prec fp32 --no-cpu-baseline --no-e2e 2>&1 | grep "debug" | tail -2; done
