"""Driver for the compute-sanitizer tier: every kernel of libhdc.so once on
small shapes (tiles, ragged tails, clusters, CTA pairs, exact cancellations that take the
recheck kernels), results checked against the oracle so a tool-induced change is visible.

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_driver.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle                                            # noqa: E402
from oracle.policy import check_fp32                     # noqa: E402
import paper_2506_09282_b200 as hdc                      # noqa: E402
from tests.gpu_util import check_result                  # noqa: E402


def run(name, prec, X, B, C, path, env=None):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        Xd, Bd, Cd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (X, B, C))
        m = hdc.Model(Bd, Cd, prec=prec)
        y, S = m.infer(Xd, path=path, return_scores=True)
        torch.cuda.synchronize()
        kernel = m.last_kernel()
        rep = check_result(prec, kernel, X, B, C, y.cpu().numpy(), S.cpu().numpy(), north_star=False)
        m.close()
        print("%-28s %-8s %-6s kernel=%-8s ok (max err/c1 %.2e)" % (name, prec, path, kernel,
                                                                  rep.get("max_err_over_c1", 0.0)), flush=True)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    rng = np.random.default_rng(0)
    N, F, D, K = 200, 150, 333, 7
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    for prec in ("fp32_tc", "bf16", "tf32"):
        run("K4 fused 2x1", prec, X, B, C, "fused")
    run("K4 fused 1x1", "bf16", X, B, C, "fused", {"HDC_TC_CLUSTER": "1x1"})
    run("K4 fused 1x2", "fp32_tc", X, B, C, "fused", {"HDC_TC_CLUSTER": "1x2"})
    run("K4 CTA pair 2x1p", "bf16", X, B, C, "fused", {"HDC_TC_CLUSTER": "2x1p"})
    run("K4 virtual 1x4", "fp32_tc", X, B, C, "fused", {"HDC_TC_CLUSTER": "1x4v"})
    run("K4 split N-tile (N=5)", "fp32_tc", X[:5], B, C, "fused")
    run("K3 fp32 FFMA", "fp32", X, B, C, "fused")
    run("K2s fp32 stream", "fp32", X[:19], B, C, "small")
    run("K2t int8 small", "fp32_tc", X[:19], B, C, "small", {"HDC_SMALL_TC": "1"})
    run("K2t int8 small (N=3)", "fp32_tc", X[:3], B, C, "small", {"HDC_SMALL_TC": "1"})
    run("K2 legacy small", "fp32", X[:9], B, C, "small", {"HDC_SMALL_LEGACY": "1"})
    # exact cancellations: the int8 recheck list and finalize kernels, K2t's recheck path
    Xi = rng.integers(-2, 3, (150, 6)).astype(np.float32)
    Bi = rng.integers(-2, 3, (6, 260)).astype(np.float32)
    Ci = rng.standard_normal((5, 260)).astype(np.float32)
    run("K4r recheck + finalize", "fp32_tc", Xi, Bi, Ci, "fused")
    run("K2t recheck", "fp32_tc", Xi[:20], Bi, Ci, "small", {"HDC_SMALL_TC": "1"})
    # encode, unfused similarity, bundling, argmax
    Bd, Cd = torch.from_numpy(B).cuda(), torch.from_numpy(C).cuda()
    m = hdc.Model(Bd, None, prec="fp32_tc", K=K)
    Hp = m.encode(torch.from_numpy(X).cuda())
    y, S = hdc.similarity_packed(Hp, D, Cd)
    labels = torch.from_numpy(rng.integers(0, K, N).astype(np.int32)).cuda()
    counts, M = hdc.bundle_classes(Hp, D, labels, K)
    am = hdc.argmax(S)
    torch.cuda.synchronize()
    orc = oracle.infer(X, B, C, allow=True)
    check_fp32(orc, y.cpu().numpy(), S.cpu().numpy())
    assert np.array_equal(am.cpu().numpy(), y.cpu().numpy())
    cnt_ref, _ = oracle.train(oracle.encode(X, B), labels.cpu().numpy(), K)
    assert np.array_equal(counts.cpu().numpy().astype(np.int64), cnt_ref)
    m.close()
    print("encode / similarity_packed / bundle / argmax ok", flush=True)
    print("SANITIZE DRIVER DONE", flush=True)


if __name__ == "__main__":
    main()
