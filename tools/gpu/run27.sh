for c in cfg3_n1 cfg3_n32; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:small --csv python bench.py --config $c --steps 3 --warmup 2 --prec fp32 --no-cpu-baseline --no-e2e 2>/dev/null | grep -v "^==" | tail -4
done
