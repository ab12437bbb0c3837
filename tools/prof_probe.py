"""Profiling probe: one model of a BASELINE config, a few inference calls (for ncu -k/-s/-c)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from hdc_inputs import CONFIGS, make_B, make_C          # noqa: E402
from hdc_inputs.device import make_X_device              # noqa: E402
import paper_2506_09282_b200 as hdc                      # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "cfg5")]
n = int(os.environ.get("NROWS", str(cfg.N)))
dev = torch.device("cuda:0")
X = make_X_device(cfg, dev, 0, n)
m = hdc.Model(torch.from_numpy(make_B(cfg)).to(dev), torch.from_numpy(make_C(cfg)).to(dev),
              prec=os.environ.get("PREC", "fp32_tc"))
for _ in range(int(os.environ.get("CALLS", "3"))):
    m.infer(X, path=os.environ.get("PATH_", "auto"))
torch.cuda.synchronize()
print("probe done", cfg.name, n, m.last_kernel())
m.close()
