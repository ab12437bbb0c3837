"""Comparison policy GPU-vs-oracle -- TEST INFRASTRUCTURE ONLY.

Implements the tolerances of BASELINE.json north_star with the readings of
DESIGN.md §3 (SURVEY.md §8c readings 10, 11):

* fp32 path: |S_gpu - S| <= 1e-4 * c1[k] + allow[n,k] for every (n, k), where
  c1[k] = ||C_k||_1 (the largest |S[n,k]| any bipolar H reaches) and allow is the
  oracle's float64-ambiguity allowance; labels identical except on rows whose
  oracle top-2 margin < 1e-4 * r[n], r[n] = max_k |S[n,k]|, where the GPU label
  must be within 1e-4 * r[n] of the oracle's best score.
* TF32/BF16 paths: |S_gpu - S| <= allow_lp[n,k] + stage2_rel(D) c1[k] always (rigorous
  allowance over the low-precision ambiguity set) and <= 1e-2 * c1[k] on the BJ configs;
  optionally fp32-policy agreement with the oracle on rounded operands; label
  agreement rate reported; every disagreement must be a near-tie at that tolerance.
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


def stage2_rel(D):
    """Rigorous relative bound of the tensor-core Stage II given exact H (T3):
    C enters as bf16 hi + lo (|c - hi - lo| <= 2^-16 |c|) and the D products accumulate
    in fp32 (gamma_tc_acc with F -> D): |S_gpu - S| <= (2^-16 + (D+1) 2^-22) ||C_k||_1."""
    return 2.0 ** -16 + (D + 1) * 2.0 ** -22


def _within(orc, y_gpu, S_gpu, tol, what):
    """Scores within the elementwise tolerance `tol` (N x K) of the oracle's, labels the
    lowest argmax of the GPU scores, and every label disagreement explained by the
    tolerance: S[n,yg] >= S[n,yo] - tol[n,yg] - tol[n,yo] (then no S inside the
    tolerances could have ranked yo strictly above yg).  Returns a report."""
    S = orc["S"]
    N, K = S.shape
    y_gpu = np.asarray(y_gpu, dtype=np.int64)
    c1 = orc["c1"]
    assert y_gpu.shape == (N,), "labels shape"
    assert np.all((y_gpu >= 0) & (y_gpu < K)), "label out of range"
    rep = {"rows": N}
    if S_gpu is not None:
        S_gpu = np.asarray(S_gpu, dtype=np.float64)
        assert S_gpu.shape == (N, K), "scores shape"
        err = np.abs(S_gpu - S)
        rep["max_err_over_c1"] = float((err / c1[None, :]).max()) if err.size else 0.0
        bad = err > tol
        rep["score_violations"] = int(bad.sum())
        assert not bad.any(), "%s: score tolerance violated at %s (err %s tol %s)" % (
            what, np.argwhere(bad)[:5].tolist(), err[bad][:5], tol[bad][:5])
        assert self_consistent(S_gpu, y_gpu), "labels are not the argmax of the GPU scores"
    agree = y_gpu == orc["y"]
    rep["agreement"] = float(agree.mean()) if N else 1.0
    rows = np.nonzero(~agree)[0]
    if rows.size:
        yo = orc["y"][rows]
        yg = y_gpu[rows]
        ok = S[rows, yg] >= S[rows, yo] - tol[rows, yg] - tol[rows, yo]
        assert ok.all(), "%s: label disagreement beyond the score tolerance at rows %s" % (
            what, rows[~ok][:10].tolist())
    return rep


def check_rounded(rounded, y_gpu, S_gpu=None, rtol=1e-4):
    """A TF32 / BF16 tensor-core result against the oracle on ROUNDED operands
    (oracle.infer(..., fmt=prec, allow=True, gamma=gamma_tc_acc(F))): the kernel must be
    the exact method on those operands up to fp32 accumulation, i.e. scores within
    rtol c1[k] (the fp32 path's 1e-4) + the accumulation allowance."""
    tol = rtol * rounded["c1"][None, :] + rounded["allow"]
    rep = _within(rounded, y_gpu, S_gpu, tol, "vs rounded operands")
    rep["amb_per_row"] = float(np.mean(rounded["namb"])) if len(rounded["namb"]) else 0.0
    return rep


def check_lowp(orc, y_gpu, S_gpu=None, rtol=1e-2, rounded=None):
    """TF32 / BF16 result against the oracle.

    orc     oracle.infer(..., allow=True, gamma=oracle.gamma_lowp(F, fmt)): the exact
            problem and its rigorous low-precision allowance.  Asserted always:
            |S_gpu - S| <= allow[n,k] + stage2_rel(D) c1[k]  (no correct kernel can exceed it).
    rtol    BASELINE north_star's 1e-2 relative to c1[k] (DESIGN reading R10), asserted
            on the BJ configs; None skips it (edge shapes whose D is too small for a
            statistical 1e-2: one flip alone moves S by 2|C[k,d]| ~ 2 c1/D).
    rounded optional oracle.infer(..., fmt=..., allow=True, gamma=gamma_tc_acc(F)) on
            the rounded operands: then check_rounded must hold as well.
    Labels: every disagreement with the exact oracle must be within the score
    tolerances (S[n,yg] >= S[n,yo] - tol[n,yg] - tol[n,yo]); agreement rates reported."""
    if orc.get("allow") is None:
        raise ValueError("check_lowp needs the oracle's low-precision allowance (allow=True)")
    c1 = orc["c1"]
    tol = orc["allow"] + stage2_rel(orc["D"]) * c1[None, :]
    if rtol is not None:
        tol = np.minimum(tol, rtol * c1[None, :])
    rep = _within(orc, y_gpu, S_gpu, tol, "vs exact (low-precision allowance)")
    rep["amb_per_row"] = float(np.mean(orc["namb"])) if len(orc["namb"]) else 0.0
    big = orc["margin"] > 2e-2 * c1.max()
    agree = np.asarray(y_gpu, dtype=np.int64) == orc["y"]
    rep["large_margin_rows"] = int(big.sum())
    rep["agreement_large_margin"] = float(agree[big].mean()) if big.any() else 1.0
    if rounded is not None:
        rep["vs_rounded"] = check_rounded(rounded, y_gpu, S_gpu)
    return rep
