"""GPU parity of the int8 tensor-core small-batch kernel K2t (k_small_tc.cu: fp32_tc
models, N <= 32) against the oracle through the C ABI, fp32 policy (sign-exact)."""
import numpy as np
import pytest
import torch

import oracle
from hdc_inputs import CONFIGS, make_B, make_C, make_X
from tests.gpu_util import parity_fp32, run_model, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _force_k2t(monkeypatch):
    monkeypatch.setenv("HDC_SMALL_TC", "1")          # K2t at every N (the default starts at 5 rows)


@pytest.fixture(scope="module")
def hdc(cuda_device):
    import paper_2506_09282_b200 as pkg
    pkg.lib()
    return pkg


def _model(hdc, B, C):
    Bd, Cd = to_dev(B, C)
    return hdc.Model(Bd, Cd, prec="fp32_tc")


@pytest.mark.parametrize("name", ["cfg3_n1", "cfg3_n4", "cfg3_n16", "cfg3_n32"])
def test_cfg3_every_row(hdc, name):
    cfg = CONFIGS[name]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    m = _model(hdc, B, C)
    rep, y, S, orc = parity_fp32(X, B, C, path="small", prec="fp32_tc", model=m)
    assert m.last_kernel() == "small_tc"
    y2, S2 = run_model(m, X, "small")
    assert np.array_equal(S, S2) and np.array_equal(y, y2)          # bit-deterministic
    m.close()
    print(name, rep)


@pytest.mark.parametrize("N,F,D,K", [
    (1, 1, 1, 1), (1, 7, 16, 2), (2, 1, 513, 2), (5, 64, 67, 3), (16, 129, 148, 26), (17, 200, 1000, 32),
    (31, 7, 17, 6), (32, 784, 10000, 10), (32, 1100, 3001, 5), (9, 3072, 2000, 10), (3, 561, 20000, 6),
    (12, 100, 149, 1)])
def test_edge_grid(hdc, N, F, D, K):
    rng = np.random.default_rng(N * 7919 + F * 101 + D * 13 + K)
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    m = _model(hdc, B, C)
    rep, y, S, orc = parity_fp32(X, B, C, path="small", prec="fp32_tc", model=m)
    kernel = m.last_kernel()
    m.close()
    assert kernel == "small_tc"
    if K == 1:
        assert np.all(y == 0)
    print((N, F, D, K), rep)


def test_exact_cancellations_zero_rows_and_duplicates(hdc):
    # integer data: exact zero pre-activations must be re-evaluated and map to +1
    rng = np.random.default_rng(17)
    X = rng.integers(-2, 3, (20, 6)).astype(np.float32)
    X[3] = 0.0
    X[4] = -0.0
    B = rng.integers(-2, 3, (6, 500)).astype(np.float32)
    C = rng.standard_normal((7, 500)).astype(np.float32)
    C[5] = C[2]
    m = _model(hdc, B, C)
    n0 = m.recheck_count()
    rep, y, S, orc = parity_fp32(X, B, C, path="small", prec="fp32_tc", model=m)
    assert m.last_kernel() == "small_tc"
    V = oracle.preact(X, B)
    assert m.recheck_count() - n0 >= int(np.sum((V == 0) & (np.abs(X).sum(1)[:, None] > 0)))
    np.testing.assert_allclose(S[3], C.astype(np.float64).sum(axis=1), rtol=1e-5, atol=1e-4)
    assert np.array_equal(S[3], S[4]) and not np.any(y == 5)
    m.close()


def test_same_labels_as_fp32_streaming_kernel(hdc, monkeypatch):
    # both kernels are sign-exact: identical H, so identical labels wherever the oracle's
    # top-2 margin is clear of fp32 rounding; scores agree to fp32 summation order
    cfg = CONFIGS["cfg3_n32"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    m = _model(hdc, B, C)
    yt, St = run_model(m, X, "small")
    monkeypatch.setenv("HDC_SMALL_TC", "0")
    ys, Ss = run_model(m, X, "small")
    assert m.last_kernel() == "small"
    m.close()
    orc = oracle.infer(X, B, C)
    clear = orc["margin"] > 1e-4 * orc["rowscale"]
    assert np.array_equal(yt[clear], ys[clear])
    assert np.max(np.abs(St - Ss)) < 1e-5 * orc["c1"].max()


def test_row_independence_and_scaling(hdc):
    # a row's labels do not depend on the batch it is in (rows are independent),
    # and X -> 2X leaves H, hence S, bit-identical (the limb image is scale-invariant)
    cfg = CONFIGS["cfg3_n32"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    m = _model(hdc, B, C)
    y32, S32 = run_model(m, X, "small")
    for n in (1, 7, 16, 17):
        yn, Sn = run_model(m, X[:n], "small")
        assert np.array_equal(yn, y32[:n])
        np.testing.assert_allclose(Sn, S32[:n], rtol=0, atol=1e-5)
    y2, S2 = run_model(m, X * np.float32(2.0), "small")
    assert np.array_equal(S2, S32) and np.array_equal(y2, y32)
    m.close()
