"""K2s with B streamed as its bf16 hi plane (sign-exact calls; k_smallstream.cu HALF):
every |v_hi| <= tau is re-evaluated in float64 and a changed sign corrects the exact
int64 score sums by (h - h_hi) C[k][d].  Judged against the oracle with the fp32 policy
(oracle/policy.py); the fp32-B stream (HDC_SMALL_FULLB) is the comparison."""
import os

import numpy as np
import pytest

import oracle
from oracle.policy import check_fp32
from hdc_inputs import CONFIGS, make_B, make_C, make_X
from tests.gpu_util import run_model, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _fp32_on_ffma(monkeypatch):
    # fp32 models stay on the fp32 kernels at every N <= 32 (K2s, not the int8 K2t)
    monkeypatch.setenv("HDC_FP32_FFMA", "1")
    monkeypatch.delenv("HDC_SMALL_FULLB", raising=False)


@pytest.fixture(scope="module")
def hdc(cuda_device):
    import paper_2506_09282_b200 as pkg
    pkg.lib()
    return pkg


def _run(m, X, fullb):
    if fullb:
        os.environ["HDC_SMALL_FULLB"] = "1"
    try:
        n0 = m.recheck_count()
        y, S = run_model(m, X, path="small")
        return y, S, m.recheck_count() - n0
    finally:
        os.environ.pop("HDC_SMALL_FULLB", None)


@pytest.mark.parametrize("name", ["cfg3_n1", "cfg3_n4", "cfg3_n16", "cfg3_n32"])
def test_cfg3_hi_plane_vs_oracle(hdc, name):
    cfg = CONFIGS[name]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    orc = oracle.infer(X, B, C, allow=True, nthreads=0)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec="fp32")
    y, S, nh = _run(m, X, fullb=False)
    assert m.last_kernel() == "small"
    rep = check_fp32(orc, y, S)
    assert rep["score_violations"] == 0
    assert np.array_equal(y, orc["y"])
    yf, Sf, nf = _run(m, X, fullb=True)
    check_fp32(orc, yf, Sf)
    # the hi plane (N = 1) has a bound ~||b_lo|| / (tau_F ||b||) ~ 10^3 times wider: many more rechecks,
    # same signs; from 2 rows K2s streams the fp32 B
    if cfg.N == 1:
        assert nh > 4 * nf
    else:
        assert nh == nf
    assert np.array_equal(y, yf)
    np.testing.assert_allclose(S, Sf, rtol=0, atol=1e-6 * np.abs(C).sum(1).max())
    m.close()


def test_rows_independent_of_batch(hdc):
    """H is exact and the flip corrections are order-free integer sums, so a row's scores
    do not depend on the rows it is batched with (bitwise) -- within one B stream: the hi
    plane (N = 1) and the fp32 B (N >= 2) differ in Stage II's fp32 rounding only."""
    cfg = CONFIGS["cfg3_n32"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec="fp32")
    y4, S4, _ = _run(m, X[:4], fullb=False)
    for n in range(4):
        y1, S1, _ = _run(m, X[n:n + 1], fullb=True)        # N = 1 on the fp32 B stream
        assert np.array_equal(S1[0], S4[n]) and y1[0] == y4[n]
        y1h, S1h, _ = _run(m, X[n:n + 1], fullb=False)     # and on the hi plane
        assert y1h[0] == y4[n]
        np.testing.assert_allclose(S1h[0], S4[n], rtol=0, atol=1e-6 * np.abs(C).sum(1).max())
    y, S, _ = _run(m, X, fullb=False)
    y8, S8, _ = _run(m, X[8:16], fullb=False)
    assert np.array_equal(S8, S[8:16]) and np.array_equal(y8, y[8:16])
    m.close()


@pytest.mark.parametrize("N", [1, 4, 32])
def test_near_zero_preactivations_flip(hdc, N):
    """Pre-activations of ~1e-7 |v| (inside the hi plane's error and the fp32 bound): every
    element is flagged and re-evaluated; on the hi plane (N = 1) the provisional signs are
    wrong about half the time and every one must be corrected (16 rows in shared-memory
    slots, the rest from L2); at N = 4 / 32 (fp32 B) the flags overflow the slots and, at
    N = 32, the CTA's deferred list (256), so the L2 and the immediate recheck paths run."""
    rng = np.random.default_rng(11 + N)
    F, D, K = 64, 2000, 5
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    X[:, F - 1] = 1.0
    B = rng.standard_normal((F, D)).astype(np.float32)
    # one shared last row cannot cancel every sample's sum: cancel sample 0's, and make
    # the other samples' last-feature weight cancel theirs (x[n, F-2] absorbs the rest)
    part = X[0, :F - 1].astype(np.float64) @ B[:F - 1].astype(np.float64)
    B[F - 1] = (-part + rng.uniform(-1e-6, 1e-6, D)).astype(np.float32)
    for n in range(1, N):
        X[n] = X[0]
        X[n, 0] = np.float32(X[0, 0] * (1 + 2.0 ** -20 * n))   # tiny, distinct perturbations
    C = rng.standard_normal((K, D)).astype(np.float32)
    V = oracle.preact(X, B)
    assert np.median(np.abs(V)) < 1e-4
    orc = oracle.infer(X, B, C, allow=True, nthreads=0)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec="fp32")
    y, S, nh = _run(m, X, fullb=False)
    rep = check_fp32(orc, y, S)
    assert rep["score_violations"] == 0
    assert nh >= int(np.sum(np.abs(V) < 1e-4))
    # the provisional bf16-B signs disagree with the exact ones on many elements
    vh = X.astype(np.float64) @ B.astype(np.float32).view(np.uint32).__and__(0xFFFF0000).view(np.float32).astype(np.float64)
    assert np.sum((vh >= 0) != (V >= 0)) > 0.1 * V.size
    m.close()
