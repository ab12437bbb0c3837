"""Degenerate inputs through every precision and path: an empty batch, a single class, a
single feature and a single column, and all-zero rows (V = 0 -> HardSign +1, so
S[n, k] = sum_d C[k, d] exactly as the oracle computes it)."""
import numpy as np
import pytest
import torch

import oracle
from tests.gpu_util import check_result, run_model, to_dev

pytestmark = pytest.mark.gpu
PRECS = ["fp32", "fp32_tc", "tf32", "bf16"]


@pytest.fixture(scope="module")
def hdc(cuda_device):
    import paper_2506_09282_b200 as pkg
    pkg.lib()
    return pkg


@pytest.mark.parametrize("prec", PRECS)
def test_empty_batch(hdc, prec):
    rng = np.random.default_rng(1)
    B = rng.standard_normal((20, 300)).astype(np.float32)
    C = rng.standard_normal((4, 300)).astype(np.float32)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec=prec)
    X = torch.empty(0, 20, dtype=torch.float32, device="cuda")
    for path in ("auto", "small", "fused"):
        y, S = m.infer(X, path=path, return_scores=True)
        assert y.shape == (0,) and S.shape == (0, 4)
    yh = torch.empty(0, dtype=torch.int32).pin_memory()
    m.infer_host(torch.empty(0, 20, dtype=torch.float32).pin_memory(), yh)
    torch.cuda.synchronize()
    if prec != "fp32":
        assert m.encode(X).shape == (0, (300 + 31) // 32)
    m.close()


def _check(prec, kernel, X, B, C, y, S):
    return check_result(prec, kernel, X, B, C, y, S, north_star=False)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("N,F,D,K", [(40, 1, 500, 3), (40, 30, 1, 3), (50, 17, 700, 1), (1, 1, 1, 1)])
def test_tiny_dimensions(hdc, prec, N, F, D, K):
    rng = np.random.default_rng(N + F + D + K)
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec=prec)
    for path in ("small", "fused"):
        y, S = run_model(m, X, path)
        rep = _check(prec, m.last_kernel(), X, B, C, y, S)
        if K == 1:
            assert np.all(y == 0)
        print(prec, path, (N, F, D, K), rep)
    m.close()


@pytest.mark.parametrize("prec", PRECS)
def test_all_zero_rows(hdc, prec):
    rng = np.random.default_rng(3)
    N, F, D, K = 70, 45, 900, 6
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    X[::7] = 0.0
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec=prec)
    y, S = run_model(m, X, "auto")
    kernel = m.last_kernel()
    m.close()
    rowsum = C.astype(np.float64).sum(axis=1)
    np.testing.assert_allclose(S[::7], np.broadcast_to(rowsum, S[::7].shape), rtol=1e-5,
                               atol=1e-4 * np.abs(C).sum(axis=1).max())
    assert np.all(y[::7] == int(np.argmax(rowsum)))
    _check(prec, kernel, X, B, C, y, S)
