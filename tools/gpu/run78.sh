mkdir -p gpurun_out
for P in bf16 fp32_tc; do
PREC=$P NROWS=2048 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r78_$P.csv python tools/small_n_probe.py > /dev/null 2>&1
done
