"""Diagnostics: dominant-kernel time of K4 under HDC_TC_DEBUG ablation flags.
The flags act only in the diagnostics build (HDC_BUILD_TAG=diag HDC_NVCC_DEFS=-DHDC_TC_DIAG=1
python -m paper_2506_09282_b200.build; run with HDC_LIB_PATH=.../lib/libhdc_diag.so)
(1 = no Stage I MMA, 2 = no operand TMA, 8 = no Stage II MMA, 16 = no epilogue
TMEM reads, 32 = Stage II only at tile boundaries).  Results of ablated runs are
wrong by construction; only their timing is of interest."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from hdc_inputs import CONFIGS, make_B, make_C          # noqa: E402
from hdc_inputs.device import make_X_device              # noqa: E402
import paper_2506_09282_b200 as hdc                      # noqa: E402


def main():
    cfg = CONFIGS[os.environ.get("CFG", "cfg2")]
    precs = os.environ.get("PRECS", "fp32_tc,bf16").split(",")
    flags = [int(f) for f in os.environ.get("FLAGS", "0,8,32,1,2,16,9").split(",")]
    dev = torch.device("cuda:0")
    X = make_X_device(cfg, dev, 0, int(os.environ.get("NROWS", cfg.N)))
    B = torch.from_numpy(make_B(cfg)).to(dev)
    C = torch.from_numpy(make_C(cfg)).to(dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    shapes = os.environ.get("SHAPES", "").split(",") if os.environ.get("SHAPES") else [None]
    for prec, shape in [(pr, sh) for pr in precs for sh in shapes]:
        if shape:
            os.environ["HDC_TC_CLUSTER"] = shape
        m = hdc.Model(B, C, prec=prec)
        m.set_kernel_timing(True)
        for fl in flags:
            os.environ["HDC_TC_DEBUG"] = str(fl)
            ts = []
            for i in range(8):
                flush.fill_(float(i))
                m.infer(X, path="fused")
                ts.append(m.last_kernel_ms())
            ts = sorted(ts[2:])
            if fl == 0:
                n0 = m.recheck_count()
                m.infer(X, path="fused")
                print("  rechecks per launch: %d" % (m.recheck_count() - n0))
            print("%s %-8s cluster=%s debug=%-3d kernel_ms median %.4f min %.4f" % (cfg.name, prec, shape, fl, ts[len(ts) // 2], ts[0]), flush=True)
        os.environ["HDC_TC_DEBUG"] = "0"
        m.close()


if __name__ == "__main__":
    main()
