"""GPU parity of the fused large-batch kernels against the oracle (C ABI).

Small shapes: every output compared.  BASELINE.json full sizes (cfg2, cfg4,
cfg5 and its D variants) run whole on the GPU in bench.py's configuration; the
oracle checks a deterministic row sample (first, last and Philox-chosen rows)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from hdc_inputs import CONFIGS, make_B, make_C, make_X
from hdc_inputs.philox import uniform_u32
from tests.gpu_util import check_result, parity_fp32, run_model, to_dev

pytestmark = pytest.mark.gpu

@pytest.fixture(autouse=True)
def _fp32_on_ffma(monkeypatch):
    # fp32 models in this module exercise the fp32 FFMA kernels (HDC_PREC_FP32 otherwise
    # runs on the int8 tensor-core kernels when eligible, tested elsewhere)
    monkeypatch.setenv("HDC_FP32_FFMA", "1")



@pytest.fixture(scope="module")
def hdc(cuda_device):
    import paper_2506_09282_b200 as pkg
    pkg.lib()
    return pkg


def sample_rows(N, n_edge=64, n_rand=1920, seed=99):
    """First and last n_edge rows plus n_rand Philox-chosen rows (2048 in total for the
    large configs, SURVEY §8d verification coverage)."""
    r = uniform_u32(seed, 7, 0, n_rand).astype(np.int64) % N
    rows = np.unique(np.concatenate([np.arange(min(n_edge, N)), np.arange(max(0, N - n_edge), N), r]))
    return rows


@pytest.mark.parametrize("N,F,D,K", [
    (33, 7, 17, 2), (127, 1, 1, 1), (128, 617, 129, 26), (129, 64, 256, 256),
    (300, 561, 2000, 6), (257, 3072, 300, 10), (200, 100, 16, 100), (1000, 33, 1000, 3)])
def test_fused_edge_grid(hdc, N, F, D, K):
    rng = np.random.default_rng(N * 7919 + F * 31 + D * 3 + K)
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    parity_fp32(X, B, C, path="fused")


def test_fused_cfg1_matches_small_path(hdc):
    cfg = CONFIGS["cfg1"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd)
    rep, yf, Sf, orc = parity_fp32(X, B, C, path="fused", model=m)
    ys, Ss = run_model(m, X, "small")
    # both sign-exact: identical H, so identical labels; scores equal up to fp32 order
    assert np.array_equal(yf, ys)
    assert np.max(np.abs(Sf - Ss)) < 1e-4
    m.close()


def test_fused_zero_rows_and_duplicates(hdc):
    rng = np.random.default_rng(3)
    X = rng.uniform(-1, 1, (200, 40)).astype(np.float32)
    X[5] = 0.0
    X[150] = -0.0
    B = rng.standard_normal((40, 500)).astype(np.float32)
    C = rng.standard_normal((7, 500)).astype(np.float32)
    C[4] = C[2]
    rep, y, S, orc = parity_fp32(X, B, C, path="fused")
    assert np.array_equal(S[5], S[150]) and not np.any(y == 4)


def test_fused_exact_cancellations(hdc):
    rng = np.random.default_rng(4)
    X = rng.integers(-2, 3, (160, 6)).astype(np.float32)
    B = rng.integers(-2, 3, (6, 300)).astype(np.float32)
    C = rng.standard_normal((5, 300)).astype(np.float32)
    parity_fp32(X, B, C, path="fused")


def test_fused_deterministic_and_metamorphic(hdc):
    cfg = CONFIGS["cfg1"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd)
    y1, S1 = run_model(m, X, "fused")
    y2, S2 = run_model(m, X, "fused")
    assert np.array_equal(S1, S2) and np.array_equal(y1, y2)
    y3, S3 = run_model(m, X * np.float32(0.5), "fused")
    assert np.array_equal(S3, S1) and np.array_equal(y3, y1)
    p = np.random.default_rng(0).permutation(X.shape[0])
    y4, S4 = run_model(m, X[p], "fused")
    assert np.array_equal(y4, y1[p])
    m.close()


def _full_size(hdc, name, prec="fp32", all_rows=None):
    """The BASELINE config run whole on the GPU (bench.py's launch configuration); the
    oracle checks every row when the config is small enough to finish in seconds (cfg1,
    cfg2, cfg3) or ``all_rows``, else the deterministic row sample (sample_rows)."""
    cfg = CONFIGS[name]
    from hdc_inputs.device import make_X_device
    B, C = make_B(cfg), make_C(cfg)
    Bd, Cd = to_dev(B, C)
    Xd = make_X_device(cfg, torch.device("cuda:0"))
    m = hdc.Model(Bd, Cd, prec=prec)
    y, S = m.infer(Xd, return_scores=True)
    torch.cuda.synchronize()
    kernel = m.last_kernel()
    y, S = y.cpu().numpy(), S.cpu().numpy()
    assert np.all((y >= 0) & (y < cfg.K))
    assert np.array_equal(np.argmax(S, axis=1), y)          # self-consistency, all rows
    if all_rows is None:
        all_rows = cfg.N <= 16384
    rows = np.arange(cfg.N) if all_rows else sample_rows(cfg.N)
    Xs = make_X(cfg) if all_rows else np.concatenate([make_X(cfg, int(r), int(r) + 1) for r in rows])
    rep = check_result(prec, kernel, Xs, B, C, y[rows], S[rows])
    rep["kernel"] = kernel
    rep["checked_rows"] = int(len(rows))
    m.close()
    out = os.environ.get("HDC_REPORT_JSONL")           # optional record for DESIGN §11 tables
    if out:
        with open(out, "a") as f:
            f.write(json.dumps({"config": name, "prec": prec, **rep}) + "\n")
    return rep


def test_cfg2_full_size(hdc):
    _full_size(hdc, "cfg2")


@pytest.mark.parametrize("name", ["cfg4", "cfg5", "cfg5_d2000", "cfg5_d20000"])
def test_large_configs_full_size(hdc, name):
    _full_size(hdc, name)
