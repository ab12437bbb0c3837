HDC_LIB_PATH=paper_2506_09282_b200/lib/libhdc_diag.so FS=128,640 FLAGS=4 PRECS=fp32_tc,bf16 timeout 300 python tools/tile_overhead.py 2>&1 | grep -v "^$" | sort | uniq -c | sort -rn | head -8
