mkdir -p gpurun_out
for P in bf16 fp32_tc; do for n in 2048 4096; do
PREC=$P NROWS=$n timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r81_${P}_$n.csv python tools/small_n_probe.py > /dev/null 2>&1
done; done
NROWS=2048 HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so FLAGS=0,4 PRECS=bf16,fp32_tc timeout 120 python tools/tc_timing.py 2>&1 | grep -v "rechecks" | sort | uniq -c | sort -rn | head -6
