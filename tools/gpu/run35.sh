mkdir -p gpurun_out/r35
timeout 600 python bench.py > gpurun_out/r35/bench_default.json 2> gpurun_out/r35/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r35/bench_ref.json 2> gpurun_out/r35/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r35/launches_cfg2_fp32_tc.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r35/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_tc --launch-skip 2 --launch-count 1 -o gpurun_out/r35/full_fused_tc_int8_cfg2 -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r35/ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_tc --launch-skip 2 --launch-count 1 -o gpurun_out/r35/full_fused_tc_bf16_cfg2 -f python bench.py --steps 2 --warmup 1 --prec bf16 --no-cpu-baseline --no-e2e > gpurun_out/r35/ncu_full_bf16.log 2>&1; echo "ncu3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smallstream --launch-skip 2 --launch-count 1 -o gpurun_out/r35/full_smallstream_cfg3_n1 -f python bench.py --config cfg3_n1 --prec fp32 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r35/ncu_full_small.log 2>&1; echo "ncu4 rc=$?"
cat gpurun_out/r35/bench_default.json; cat gpurun_out/r35/bench_ref.json
