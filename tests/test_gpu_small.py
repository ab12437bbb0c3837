"""GPU parity of the small-batch D-split kernel (K2) against the oracle, through
the C ABI.  fp32 tolerance policy: oracle/policy.py."""
import numpy as np
import pytest
import torch

import oracle
from hdc_inputs import CONFIGS, make_B, make_C, make_X
from tests.gpu_util import parity_fp32, run_model, to_dev

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


@pytest.mark.parametrize("name", ["cfg3_n1", "cfg3_n4", "cfg3_n16", "cfg3_n32"])
def test_cfg3_small_batch(hdc, name):
    cfg = CONFIGS[name]
    rep, y, S, orc = parity_fp32(make_X(cfg), make_B(cfg), make_C(cfg), path="small")
    assert rep["score_violations"] == 0


def test_cfg1_full(hdc):
    cfg = CONFIGS["cfg1"]
    rep, *_ = parity_fp32(make_X(cfg), make_B(cfg), make_C(cfg), path="small")
    assert rep["rows"] == 256


@pytest.mark.parametrize("N,F,D,K", [
    (1, 1, 1, 1), (1, 7, 16, 2), (31, 7, 17, 6), (32, 129, 33, 26), (33, 64, 300, 3),
    (5, 561, 1000, 256), (3, 3072, 257, 10), (2, 1, 513, 2), (17, 200, 31, 100)])
def test_edge_grid(hdc, N, F, D, K):
    rng = np.random.default_rng(N * 1000003 + F * 1009 + D * 7 + K)
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    parity_fp32(X, B, C, path="small")


def test_zero_rows_negzero_duplicate_classes(hdc):
    rng = np.random.default_rng(5)
    X = rng.uniform(-1, 1, (9, 50)).astype(np.float32)
    X[0] = 0.0
    X[1] = -0.0
    B = rng.standard_normal((50, 700)).astype(np.float32)
    C = rng.standard_normal((5, 700)).astype(np.float32)
    C[3] = C[1]
    rep, y, S, orc = parity_fp32(X, B, C, path="small")
    assert np.all(S[0] == S[1])
    np.testing.assert_allclose(S[0], C.astype(np.float64).sum(axis=1), rtol=1e-5, atol=1e-4)
    assert not np.any(y == 3)          # duplicate class never beats its lower twin


def test_exact_cancellations_are_rechecked(hdc):
    """Integer data with exact zero pre-activations: HardSign(0) = +1 must hold
    and the fp64 re-evaluation path must run (rows with V == 0, W > 0)."""
    rng = np.random.default_rng(6)
    X = rng.integers(-2, 3, (8, 6)).astype(np.float32)
    B = rng.integers(-2, 3, (6, 400)).astype(np.float32)
    C = rng.standard_normal((4, 400)).astype(np.float32)
    import paper_2506_09282_b200 as pkg
    Bd, Cd = to_dev(B, C)
    m = pkg.Model(Bd, Cd)
    before = m.recheck_count()
    rep, y, S, orc = parity_fp32(X, B, C, path="small", model=m)
    V = oracle.preact(X, B)
    assert m.recheck_count() - before >= int(np.sum(V == 0))
    m.close()


def test_deterministic_and_scaling_invariant(hdc):
    cfg = CONFIGS["cfg3_n16"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd)
    y1, S1 = run_model(m, X, "small")
    y2, S2 = run_model(m, X, "small")
    assert np.array_equal(S1, S2) and np.array_equal(y1, y2)
    y3, S3 = run_model(m, X * np.float32(8.0), "small")      # H unchanged -> bitwise
    assert np.array_equal(S3, S1) and np.array_equal(y3, y1)
    y4, S4 = run_model(m, -X, "small")                         # X -> -X: V -> -V exactly
    if not np.any(oracle.preact(X, B) == 0):
        assert np.array_equal(S4, -S1)
    m.close()
    Cd2 = to_dev(C * np.float32(0.25))[0]
    m2 = hdc.Model(Bd, Cd2)
    y5, S5 = run_model(m2, X, "small")
    assert np.array_equal(S5, S1 * np.float32(0.25)) and np.array_equal(y5, y1)
    m2.close()


def test_oneshot_host_and_partial_scores(hdc):
    cfg = CONFIGS["cfg3_n4"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    Xd, Bd, Cd = to_dev(X, B, C)
    m = hdc.Model(Bd, Cd)
    y, S = run_model(m, X, "small")
    y1, S1 = hdc.infer(Xd, Bd, Cd, return_scores=True)
    torch.cuda.synchronize()
    assert np.array_equal(y1.cpu().numpy(), y) and np.array_equal(S1.cpu().numpy(), S)
    # host-buffer (e2e) entry point
    Xh = torch.from_numpy(X).pin_memory()
    yh = torch.empty(X.shape[0], dtype=torch.int32).pin_memory()
    Sh = torch.empty(X.shape[0], cfg.K, dtype=torch.float32).pin_memory()
    m.infer_host(Xh, yh, Sh)
    torch.cuda.synchronize()
    assert np.array_equal(yh.numpy(), y) and np.array_equal(Sh.numpy(), S)
    # D-split partial scores (Alg. 3 S += S_local): sum of two halves ~ full
    cut = 4992
    ma = hdc.Model(Bd[:, :cut].contiguous(), Cd[:, :cut].contiguous())
    mb = hdc.Model(Bd[:, cut:].contiguous(), Cd[:, cut:].contiguous())
    Ssum = (ma.partial_scores(Xd) + mb.partial_scores(Xd))
    lab = hdc.argmax(Ssum)
    torch.cuda.synchronize()
    orc = oracle.infer(X, B, C, allow=True)
    from oracle.policy import check_fp32
    check_fp32(orc, lab.cpu().numpy(), Ssum.cpu().numpy())
    for mm in (m, ma, mb):
        mm.close()


def test_argmax_ties_lowest_index(hdc):
    S = torch.tensor([[0.1, 3.0, -1.0, 3.0], [2.0, 2.0, 2.0, 2.0], [-5.0, -4.0, -4.0, -6.0]],
                     device="cuda")
    assert hdc.argmax(S).cpu().tolist() == [1, 0, 1]
    S2 = torch.randn(1000, 300, device="cuda")
    S2[:, 7] = S2.max(dim=1).values
    S2[:, 250] = S2[:, 7]
    assert np.array_equal(hdc.argmax(S2).cpu().numpy(), np.argmax(S2.cpu().numpy(), axis=1))


@pytest.mark.parametrize("prec", ["fp32_tc", "bf16"])
def test_host_path_pipelined_calls(hdc, prec):
    # back-to-back host-buffer calls share two staging buffers and overlap the copy of
    # call i + 1 with the compute of call i; every call's labels / scores must equal the
    # device-resident call on the same rows (chunked: N > 8192; growing N reallocates;
    # a call on another stream must not race the previous call's outputs)
    rng = np.random.default_rng(5)
    F, D, K = 97, 3000, 7
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec=prec)
    sizes = [5000, 20000, 20000, 33, 20000, 30000, 7]
    Xs = [rng.uniform(-1, 1, (n, F)).astype(np.float32) for n in sizes]
    hosts = [(torch.from_numpy(X).pin_memory(), torch.empty(X.shape[0], dtype=torch.int32).pin_memory(),
              torch.empty(X.shape[0], K, dtype=torch.float32).pin_memory()) for X in Xs]
    side = torch.cuda.Stream()
    for i, (Xh, yh, Sh) in enumerate(hosts):
        m.infer_host(Xh, yh, Sh, stream=side if i == 4 else None)
    torch.cuda.synchronize()
    for X, (Xh, yh, Sh) in zip(Xs, hosts):
        y, S = run_model(m, X, "auto")
        # chunking changes how a row's D-range is split over CTAs, so the fp32 partial
        # sums may round differently; labels must agree wherever the top-2 gap is clear
        np.testing.assert_allclose(Sh.numpy(), S, rtol=1e-5, atol=1e-3)
        top2 = np.sort(S, axis=1)[:, -2:]
        clear = (top2[:, 1] - top2[:, 0]) > 1e-2
        assert np.array_equal(yh.numpy()[clear], y[clear])
    m.close()


def test_host_path_pageable_outputs(hdc):
    # non-pinned (pageable) label / score buffers take the device-to-host copy path; pinned
    # ones are written directly by the kernels -- both must give the device-call results
    rng = np.random.default_rng(9)
    F, D, K, N = 50, 1500, 5, 300
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec="fp32_tc")
    y, S = run_model(m, X, "auto")
    Xh = torch.from_numpy(X).pin_memory()
    yp, Sp = torch.empty(N, dtype=torch.int32), torch.empty(N, K, dtype=torch.float32)   # pageable
    m.infer_host(Xh, yp, Sp)
    torch.cuda.synchronize()
    np.testing.assert_allclose(Sp.numpy(), S, rtol=1e-5, atol=1e-3)
    top2 = np.sort(S, axis=1)[:, -2:]
    clear = (top2[:, 1] - top2[:, 0]) > 1e-2
    assert np.array_equal(yp.numpy()[clear], y[clear])
    m.close()
