"""Every-row parity of the large BASELINE configs (test infrastructure, run on the GPU box).

The `-m gpu` suite checks cfg4 / cfg5 on a 2048-row sample (its time budget); this tool runs
the whole batch on the GPU in bench.py's configuration and the float64 oracle on every row
(all host cores), judges it with the policy of its precision (oracle/policy.py check_fp32,
check_lowp for bf16 / tf32) and writes a
JSON report:

    python tools/full_parity.py [cfg4 cfg5:bf16 ...] > report.jsonl
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle                                            # noqa: E402
from oracle.policy import check_fp32, check_lowp         # noqa: E402
from hdc_inputs import CONFIGS, make_B, make_C, make_X   # noqa: E402
import paper_2506_09282_b200 as hdc                      # noqa: E402


def run(name, prec="fp32_tc"):
    cfg = CONFIGS[name]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    dev = torch.device("cuda:0")
    m = hdc.Model(torch.from_numpy(B).to(dev), torch.from_numpy(C).to(dev), prec=prec)
    y, S = m.infer(torch.from_numpy(X).to(dev), return_scores=True)
    torch.cuda.synchronize()
    y, S = y.cpu().numpy(), S.cpu().numpy()
    rep = {"config": name, "prec": prec, "N": int(cfg.N), "F": int(cfg.F), "D": int(cfg.D), "K": int(cfg.K),
           "kernel": m.last_kernel(), "tile_n": m.tc_tile_n()}
    m.close()
    t0 = time.time()
    if prec in ("bf16", "tf32"):
        # the low-precision policy against the exact problem (rigorous allowance, north_star's
        # 1e-2 on the BASELINE configs) and the fp32 policy against the rounded-operand problem
        exact, rounded = oracle.infer_lowp(X, B, C, prec, nthreads=0)
        rep["oracle_s"] = round(time.time() - t0, 1)
        rep.update(check_lowp(exact, y, S, rtol=1e-2, rounded=rounded))
        rep["labels_equal_oracle"] = int(np.sum(y == exact["y"]))
    else:
        orc = oracle.infer(X, B, C, allow=True, nthreads=0)
        rep["oracle_s"] = round(time.time() - t0, 1)
        rep.update(check_fp32(orc, y, S))
        rep["labels_equal_oracle"] = int(np.sum(y == orc["y"]))
    rep["verdict"] = "pass"
    return rep


if __name__ == "__main__":
    # arguments: config[:precision] ...
    names = sys.argv[1:] or ["cfg4", "cfg5"]
    out = []
    for a in names:
        n, _, p = a.partition(":")
        r = run(n, p or "fp32_tc")
        print(json.dumps(r, default=float), flush=True)
        out.append(r)
