timeout 600 python tools/tile_overhead.py 2>&1 | grep -v "^\[hdc"
