mkdir -p gpurun_out/r148
for mode in unfused train; do for pr in fp32_tc bf16; do timeout 300 python bench.py --mode $mode --prec $pr --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r148/bench_cfg2_${mode}_$pr.json 2> gpurun_out/r148/bench_cfg2_${mode}_$pr.err; echo "$mode $pr rc=$?"; done; done
