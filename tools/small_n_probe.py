"""Diagnostics: run a few fused-path inferences at a given N (for an ncu launch list)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from hdc_inputs import CONFIGS, make_B, make_C          # noqa: E402
from hdc_inputs.device import make_X_device              # noqa: E402
import paper_2506_09282_b200 as hdc                      # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "cfg2")]
n = int(os.environ.get("NROWS", "2048"))
dev = torch.device("cuda:0")
X = make_X_device(cfg, dev, 0, n)
m = hdc.Model(torch.from_numpy(make_B(cfg)).to(dev), torch.from_numpy(make_C(cfg)).to(dev),
              prec=os.environ.get("PREC", "fp32_tc"))
for _ in range(3):
    m.infer(X)
torch.cuda.synchronize()
m.close()
