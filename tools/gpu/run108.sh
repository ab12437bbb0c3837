timeout 120 python tools/symm_probe.py 2>&1 | tail -8
nvidia-smi topo -m 2>&1 | head -5
