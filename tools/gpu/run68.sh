timeout 900 python -m pytest tests/test_gpu_tc.py -x -q -k "large_configs or cfg2" 2>&1 | tail -2
for c in cfg5 cfg5_d20000 cfg5_d2000; do CFG=$c SHAPES= FLAGS=0 PRECS=fp32_tc,bf16 timeout 600 python tools/tc_timing.py 2>&1 | grep -v "^\[hdc\|rechecks" | tail -2; done
CFG=cfg5 FLAGS=0 PRECS=fp32_tc timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:fused_tc -c 1 --csv python tools/tc_timing.py 2>/dev/null | grep -o '"dram__bytes_read.sum","byte","[0-9,]*"\|"gpu__time_duration.sum","ns","[0-9,]*"'
