"""Seeded random shapes through the product entry point (path auto) against the oracle:
fp32-semantics models under the fp32 policy, tf32 / bf16 models under the low-precision
policy.  Shapes straddle every tile boundary (N-tiles of 128, D-tiles of 80 / 160, K
stages of 64 / 128 bytes, the N <= 32 small-batch kernel)."""
import numpy as np
import pytest

from tests.gpu_util import check_result, run_model, to_dev

pytestmark = pytest.mark.gpu


def _shapes(seed, n):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        N = int(rng.choice([int(rng.integers(1, 33)), int(rng.integers(33, 700))]))
        F = int(rng.integers(1, 1100))
        D = int(rng.integers(1, 3000))
        K = int(rng.integers(2, 33))
        out.append((N, F, D, K))
    return out


@pytest.fixture(scope="module")
def hdc(cuda_device):
    import paper_2506_09282_b200 as pkg
    pkg.lib()
    return pkg


@pytest.mark.parametrize("prec", ["fp32", "fp32_tc", "tf32", "bf16"])
@pytest.mark.parametrize("case", range(6))
def test_random_shapes(hdc, prec, case):
    N, F, D, K = _shapes(1234 + case, 6)[case]
    rng = np.random.default_rng(case * 977 + len(prec))
    lo = -1.0 if case % 2 else 0.0                      # both BASELINE input ranges
    X = rng.uniform(lo, 1.0, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    C /= np.linalg.norm(C.astype(np.float64), axis=1, keepdims=True).astype(np.float32)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec=prec)
    y, S = run_model(m, X, "auto")
    kernel = m.last_kernel()
    m.close()
    rep = check_result(prec, kernel, X, B, C, y, S, north_star=False)
    print(prec, (N, F, D, K), kernel, rep)
