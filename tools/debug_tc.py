"""Ad-hoc diagnostic for the tcgen05 kernel (not collected by pytest)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import oracle
import paper_2506_09282_b200 as hdc

def run(prec, N, F, D, K, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    Xd, Bd, Cd = (torch.from_numpy(a).cuda() for a in (X, B, C))
    m = hdc.Model(Bd, Cd, prec=prec)
    y, S = m.infer(Xd, path="fused", return_scores=True)
    torch.cuda.synchronize()
    orc = oracle.infer(X, B, C)
    S = S.cpu().numpy(); y = y.cpu().numpy()
    err = np.abs(S - orc["S"]) / orc["c1"][None, :]
    print(prec, (N, F, D, K), "max err/c1 %.3g" % err.max(), "agree %.4f" % (y == orc["y"]).mean(),
          "rechecks", m.recheck_count(), flush=True)
    if err.max() > 1e-2:
        print(" S[0,:4]", S[0, :4], "orc", orc["S"][0, :4])
        bad = np.argwhere(err > 1e-2)
        print(" bad rows", np.unique(bad[:, 0])[:20], "count", len(bad))

for prec in sys.argv[1:] or ["bf16", "tf32", "fp32_tc"]:
    for shp in [(128, 64, 80, 4), (128, 617, 160, 26), (300, 561, 2000, 6)]:
        run(prec, *shp)
