"""Diagnostics: small-batch latency of the small-batch kernel (K2s) vs the fused
tensor-core kernel (K4) at N = 1..32, L2 flushed before every call (bench protocol)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from hdc_inputs import CONFIGS, make_B, make_C          # noqa: E402
from hdc_inputs.device import make_X_device              # noqa: E402
import paper_2506_09282_b200 as hdc                      # noqa: E402


def main():
    cfg = CONFIGS[os.environ.get("CFG", "cfg3_n32")]
    dev = torch.device("cuda:0")
    X = make_X_device(cfg, dev, 0, 32)
    B = torch.from_numpy(make_B(cfg)).to(dev)
    C = torch.from_numpy(make_C(cfg)).to(dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for prec in os.environ.get("PRECS", "fp32_tc,bf16").split(","):
        m = hdc.Model(B, C, prec=prec)
        m.set_kernel_timing(True)
        for n in (1, 4, 16, 32):
            for path in ("small", "fused"):
                ts = []
                for i in range(12):
                    flush.fill_(float(i))
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    m.infer(X[:n], path=path)
                    e.record()
                    torch.cuda.synchronize()
                    ts.append(s.elapsed_time(e))
                ts = sorted(ts[2:])
                print("%s %-8s N=%2d %-6s call %.4f ms (min %.4f)  dominant kernel %.4f ms" %
                      (cfg.name, prec, n, path, ts[len(ts) // 2], ts[0], m.last_kernel_ms()), flush=True)
        m.close()


if __name__ == "__main__":
    main()
