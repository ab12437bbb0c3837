timeout 300 python tools/smalln_probe.py 2>&1 | grep -v "^\[hdc"
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -k "small_batch or edge_grid" 2>&1 | tail -2
