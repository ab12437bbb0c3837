"""Diagnostics: host->device copy bandwidth alone vs while the fused kernel runs on
another stream (does compute slow the PCIe DMA?)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from hdc_inputs import CONFIGS, make_B, make_C          # noqa: E402
from hdc_inputs.device import make_X_device              # noqa: E402
import paper_2506_09282_b200 as hdc                      # noqa: E402


def main():
    cfg = CONFIGS["cfg2"]
    dev = torch.device("cuda:0")
    X = make_X_device(cfg, dev, 0, cfg.N)
    m = hdc.Model(torch.from_numpy(make_B(cfg)).to(dev), torch.from_numpy(make_C(cfg)).to(dev),
                  prec=os.environ.get("PREC", "fp32_tc"))
    h = X.cpu().pin_memory()
    d = torch.empty_like(X)
    cs, ks = torch.cuda.Stream(), torch.cuda.Stream()
    for mode in ("copy alone", "compute alone", "both"):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if mode != "compute alone":
            with torch.cuda.stream(cs):
                e0.record()
                for _ in range(20):
                    d.copy_(h, non_blocking=True)
                e1.record()
        if mode != "copy alone":
            with torch.cuda.stream(ks):
                f0.record()
                for _ in range(20):
                    m.infer(X, stream=ks)
                f1.record()
        torch.cuda.synchronize()
        msg = mode
        if mode != "compute alone":
            ms = e0.elapsed_time(e1) / 20
            msg += "  copy %.3f ms (%.1f GB/s)" % (ms, h.numel() * 4 / ms / 1e6)
        if mode != "copy alone":
            msg += "  infer %.3f ms" % (f0.elapsed_time(f1) / 20)
        print(msg, flush=True)
    m.close()


if __name__ == "__main__":
    main()
