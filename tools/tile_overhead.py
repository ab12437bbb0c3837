"""Diagnostics: fused-kernel time vs K stages per tile (F sweep at fixed N, D, K) to
separate the per-stage cost from the per-tile cost (T = a * stages + b * tiles)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_09282_b200 as hdc                      # noqa: E402


def main():
    N, D, K = 16384, 10000, 26
    dev = torch.device("cuda:0")
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    for prec in os.environ.get("PRECS", "bf16,fp32_tc").split(","):
        rows = []
        for F in [int(f) for f in os.environ.get("FS", "128,256,384,512,768,1024").split(",")]:
            X = torch.rand(N, F, device=dev, generator=g) * 2 - 1
            B = torch.randn(F, D, device=dev, generator=g)
            C = torch.randn(K, D, device=dev, generator=g)
            m = hdc.Model(B, C, prec=prec)
            m.set_kernel_timing(True)
            os.environ["HDC_TC_DEBUG"] = os.environ.get("FLAGS", "0")
            ts = []
            for i in range(8):
                flush.fill_(float(i))
                m.infer(X, path="fused")
                ts.append(m.last_kernel_ms())
            m.close()
            t = sorted(ts[2:])[len(ts[2:]) // 2]
            rows.append((F, t))
            print("%s F=%5d kernel %.4f ms" % (prec, F, t), flush=True)
        F = np.array([r[0] for r in rows], dtype=np.float64)
        T = np.array([r[1] for r in rows])
        if len(F) < 2:
            continue
        a, b = np.polyfit(F, T, 1)
        print("%s fit: T = %.6f ms per 64 F + %.4f ms (F-independent)" % (prec, a * 64, b))


if __name__ == "__main__":
    main()
