"""Comparison policy GPU-vs-oracle -- TEST INFRASTRUCTURE ONLY.

Implements the tolerances of BASELINE.json north_star with the readings of
DESIGN.md §3 (SURVEY.md §8c readings 10, 11):

* fp32 path: |S_gpu - S| <= 1e-4 * c1[k] + allow[n,k] for every (n, k), where
  c1[k] = ||C_k||_1 (the largest |S[n,k]| any bipolar H reaches) and allow is the
  oracle's float64-ambiguity allowance; labels identical except on rows whose
  oracle top-2 margin < 1e-4 * r[n], r[n] = max_k |S[n,k]|, where the GPU label
  must be within 1e-4 * r[n] of the oracle's best score.
* TF32/BF16 paths: |S_gpu - S| <= 1e-2 * c1[k]; label agreement rate reported;
  every disagreement must be a near-tie at that tolerance.
* all paths: labels in [0, K); y_gpu = lowest-index argmax of S_gpu.
"""
import numpy as np


def self_consistent(S_gpu, y_gpu):
    """y must be the lowest index of the maximum of each S row (bit-exact check)."""
    S_gpu = np.asarray(S_gpu)
    if S_gpu.shape[0] == 0:
        return True
    return bool(np.array_equal(np.argmax(S_gpu, axis=1).astype(np.int32), np.asarray(y_gpu, np.int32)))


def check_fp32(orc, y_gpu, S_gpu=None, rtol=1e-4):
    S = orc["S"]
    N, K = S.shape
    y_gpu = np.asarray(y_gpu, dtype=np.int64)
    rep = {"rows": N}
    assert y_gpu.shape == (N,)
    assert np.all((y_gpu >= 0) & (y_gpu < K)), "label out of range"
    if S_gpu is not None:
        S_gpu = np.asarray(S_gpu, dtype=np.float64)
        allow = orc["allow"] if orc["allow"] is not None else np.zeros_like(S)
        tol = rtol * orc["c1"][None, :] + allow
        err = np.abs(S_gpu - S)
        rep["max_abs_err"] = float(err.max()) if err.size else 0.0
        rep["max_err_over_c1"] = float((err / orc["c1"][None, :]).max()) if err.size else 0.0
        bad = err > tol
        rep["score_violations"] = int(bad.sum())
        assert not bad.any(), "score tolerance violated at %s (err %s tol %s)" % (
            np.argwhere(bad)[:5].tolist(), err[bad][:5], tol[bad][:5])
        assert self_consistent(S_gpu, y_gpu), "labels are not the argmax of the GPU scores"
    r = orc["rowscale"]
    exempt = orc["margin"] < rtol * r
    rep["exempt_rows"] = int(exempt.sum())
    mism = (y_gpu != orc["y"])
    hard = mism & ~exempt
    assert not hard.any(), "label mismatch on non-exempt rows %s" % np.nonzero(hard)[0][:10].tolist()
    soft = mism & exempt
    if soft.any():
        rows = np.nonzero(soft)[0]
        best = S[rows].max(axis=1)
        ok = S[rows, y_gpu[rows]] >= best - rtol * r[rows]
        assert ok.all(), "exempt-row label not a near-tie"
    rep["label_mismatch"] = int(mism.sum())
    return rep


def check_lowp(orc, y_gpu, S_gpu=None, rtol=1e-2):
    S = orc["S"]
    N, K = S.shape
    y_gpu = np.asarray(y_gpu, dtype=np.int64)
    c1 = orc["c1"]
    assert np.all((y_gpu >= 0) & (y_gpu < K)), "label out of range"
    rep = {"rows": N}
    if S_gpu is not None:
        S_gpu = np.asarray(S_gpu, dtype=np.float64)
        err = np.abs(S_gpu - S)
        rep["max_err_over_c1"] = float((err / c1[None, :]).max()) if err.size else 0.0
        bad = err > rtol * c1[None, :]
        rep["score_violations"] = int(bad.sum())
        assert not bad.any(), "score tolerance violated (max err/c1 %g)" % rep["max_err_over_c1"]
        assert self_consistent(S_gpu, y_gpu), "labels are not the argmax of the GPU scores"
    agree = y_gpu == orc["y"]
    rep["agreement"] = float(agree.mean()) if N else 1.0
    big = orc["margin"] > 2e-2 * c1.max()
    rep["agreement_large_margin"] = float(agree[big].mean()) if big.any() else 1.0
    rows = np.nonzero(~agree)[0]
    if rows.size:
        yo = orc["y"][rows]
        yg = y_gpu[rows]
        ok = S[rows, yg] >= S[rows, yo] - rtol * (c1[yg] + c1[yo])
        assert ok.all(), "low-precision label disagreement beyond tolerance"
    return rep
