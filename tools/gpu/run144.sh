timeout 200 python tools/copy_interference.py 2>&1 | grep -v "^\[hdc"
PREC=bf16 timeout 200 python tools/copy_interference.py 2>&1 | grep -v "^\[hdc"
