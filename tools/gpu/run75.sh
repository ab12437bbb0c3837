# PCIe copy bandwidth (e2e bound) + CTA-pair parity tests
nvidia-smi -q | grep -i -A3 "Link Width\|PCIe Generation" | head -20
timeout 120 python tools/h2d_bw.py
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "pair" 2>&1 | tail -3
