"""GPU parity of K4's int8 "wide" mode (160-column tiles of two 80-column sub-tiles, one
accumulator buffer), the default for fp32-semantics models with K <= 16 and
padded F >= 768, forced elsewhere with HDC_TC_WIDE=1 (read at model creation).

The wide mode changes the tile width of the sign-exact Stage I and the Stage II tile sums,
not the arithmetic contract: results must meet the fp32 policy against the oracle."""
import numpy as np
import pytest

import oracle
from tests.gpu_util import parity, parity_fp32, run_model, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hdc(cuda_device):
    import paper_2506_09282_b200 as pkg
    pkg.lib()
    return pkg


def _inputs(N, F, D, K, seed):
    rng = np.random.default_rng(seed)
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    return X, B, C


@pytest.mark.parametrize("N,F,D,K", [(33, 7, 17, 2), (300, 561, 333, 7), (129, 64, 801, 16),
                                     (257, 150, 2000, 10), (200, 100, 16, 1), (1000, 33, 161, 3)])
def test_wide_forced_edge_grid(hdc, monkeypatch, N, F, D, K):
    """Ragged N / D tails, a single partial tile, D past one or several 160-column tiles."""
    monkeypatch.setenv("HDC_TC_WIDE", "1")
    X, B, C = _inputs(N, F, D, K, N * 7 + F * 3 + D + K)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec="fp32_tc")
    assert m.tc_tile_n() == 160
    rep, y, S = parity(X, B, C, path="fused", model=m, north_star=False)
    assert rep["kernel"] == "tc"
    m.close()


def test_wide_default_by_F(hdc, monkeypatch):
    """Padded F >= 768 and K <= 16 select the wide mode; K > 16 or smaller F do not."""
    monkeypatch.delenv("HDC_TC_WIDE", raising=False)
    X, B, C = _inputs(150, 2100, 500, 10, 5)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec="fp32_tc")
    assert m.tc_tile_n() == 160
    rep, y, S = parity(X, B, C, path="fused", model=m, north_star=False)
    assert rep["kernel"] == "tc"
    m.close()
    C20 = np.random.default_rng(6).standard_normal((20, 500)).astype(np.float32)
    m = hdc.Model(Bd, to_dev(C20)[0], prec="fp32_tc")
    assert m.tc_tile_n() == 80
    m.close()
    m = hdc.Model(*to_dev(B[:700], C), prec="fp32_tc")
    assert m.tc_tile_n() == 80
    m.close()
    monkeypatch.setenv("HDC_TC_WIDE", "0")
    m = hdc.Model(Bd, Cd, prec="fp32_tc")
    assert m.tc_tile_n() == 80
    m.close()


def test_wide_exact_cancellations(hdc, monkeypatch):
    """Integer inputs with exact zero pre-activations: the coarse flag test must still list
    every |I| <= tau element (the fp64 recheck then fixes the signs)."""
    monkeypatch.setenv("HDC_TC_WIDE", "1")
    rng = np.random.default_rng(11)
    X = rng.integers(-2, 3, (300, 6)).astype(np.float32)
    X[7] = 0.0
    B = rng.integers(-2, 3, (6, 400)).astype(np.float32)
    C = rng.standard_normal((5, 400)).astype(np.float32)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec="fp32_tc")
    assert m.tc_tile_n() == 160
    n0 = m.recheck_count()
    rep, y, S, orc = parity_fp32(X, B, C, path="fused", prec="fp32_tc", model=m)
    V = oracle.preact(X, B)
    assert m.recheck_count() - n0 >= int(np.sum((V == 0) & (np.abs(X).sum(1)[:, None] > 0)))
    m.close()


def test_wide_encode_matches_oracle(hdc, monkeypatch):
    """Encode mode (bit-packed H) of the wide kernel: every sign equals the oracle's."""
    monkeypatch.setenv("HDC_TC_WIDE", "1")
    X, B, C = _inputs(200, 300, 500, 4, 9)
    Bd, = to_dev(B)
    m = hdc.Model(Bd, None, prec="fp32_tc", K=4)
    assert m.tc_tile_n() == 160
    (Xd,) = to_dev(X)
    Hp = m.encode(Xd)
    H = hdc.unpack_signs(Hp, 500).cpu().numpy()
    assert np.array_equal(H, oracle.encode(X, B))
    m.close()


def test_wide_deterministic_and_n_invariant(hdc, monkeypatch):
    """Exact int64 Stage II sums: bitwise identical scores for a row however the batch is cut."""
    monkeypatch.setenv("HDC_TC_WIDE", "1")
    X, B, C = _inputs(700, 200, 900, 8, 13)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec="fp32_tc")
    y1, S1 = run_model(m, X, "fused")
    y2, S2 = run_model(m, X, "fused")
    assert np.array_equal(S1, S2) and np.array_equal(y1, y2)
    y3, S3 = run_model(m, X[300:], "fused")
    assert np.array_equal(S3, S1[300:]) and np.array_equal(y3, y1[300:])
    m.close()
