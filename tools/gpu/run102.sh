timeout 300 python tools/smalln_probe.py 2>&1 | grep -v "^\[hdc"
