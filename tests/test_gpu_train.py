"""GPU parity of the materialised-H entry points against the oracle, via the C ABI:
hdc_model_encode (Stage I alone, bit-packed H), hdc_similarity_packed (the unfused
Stage II of the fusion ablation) and hdc_bundle_classes (single-pass training).

fp32_tc encoding is sign-exact -> H, the class counts and M must equal the oracle's
bit for bit; bf16/tf32 encodings may flip signs only where |V| is within the
low-precision rounding of the product (checked element by element)."""
import numpy as np
import pytest
import torch

import oracle
from oracle.policy import check_fp32
from hdc_inputs import CONFIGS, make_B, make_C, make_X
from tests.gpu_util import to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hdc(cuda_device):
    import paper_2506_09282_b200 as pkg
    pkg.lib()
    return pkg


def _unpack(hdc, H, D):
    return hdc.unpack_signs(H, D).cpu().numpy().astype(np.int8)


SHAPES = [(33, 7, 17), (128, 617, 160), (129, 64, 250), (300, 561, 2000), (257, 3072, 300),
          (200, 100, 16), (1000, 33, 1000), (640, 784, 801), (1, 1, 1), (130, 40, 2001)]


@pytest.mark.parametrize("N,F,D", SHAPES)
def test_encode_fp32_tc_exact(hdc, N, F, D):
    rng = np.random.default_rng(N * 7 + F * 3 + D)
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    Bd, = to_dev(B)
    m = hdc.Model(Bd, None, prec="fp32_tc", K=1)
    H = m.encode(torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    m.close()
    assert H.shape == (N, (D + 31) // 32)
    Hg = _unpack(hdc, H, D)
    Ho = oracle.encode(X, B)
    assert np.array_equal(Hg, Ho), "sign mismatches: %d" % int(np.sum(Hg != Ho))
    # bits past D stay clear
    if D % 32:
        assert int(torch.sum((H[:, -1] >> (D % 32)) != 0)) == 0


def test_encode_exact_cancellations(hdc):
    rng = np.random.default_rng(4)
    X = rng.integers(-2, 3, (300, 6)).astype(np.float32)
    X[5] = 0.0
    B = rng.integers(-2, 3, (6, 400)).astype(np.float32)
    m = hdc.Model(torch.from_numpy(B).cuda(), None, prec="fp32_tc", K=1)
    Hg = _unpack(hdc, m.encode(torch.from_numpy(X).cuda()), 400)
    m.close()
    assert np.array_equal(Hg, oracle.encode(X, B))        # V = 0 -> +1


@pytest.mark.parametrize("prec", ["bf16", "tf32"])
def test_encode_lowp_flips_only_near_zero(hdc, prec):
    cfg = CONFIGS["cfg1"]
    X, B = make_X(cfg, 0, 128), make_B(cfg)
    m = hdc.Model(torch.from_numpy(B).cuda(), None, prec=prec, K=1)
    Hg = _unpack(hdc, m.encode(torch.from_numpy(X).cuda()), cfg.D)
    m.close()
    V = oracle.preact(X, B)
    W = np.abs(X).astype(np.float64) @ np.abs(B).astype(np.float64)
    u = 2.0 ** -8 if prec == "bf16" else 2.0 ** -11       # unit roundoff of the staged operands
    bound = ((2 * u + u * u) + (cfg.F + 2) * 2.0 ** -24) * W * 1.01 + 1e-30   # operands + fp32 accumulation
    flips = Hg != oracle.encode(X, B)
    print(prec, "flips", int(flips.sum()), "of", flips.size)
    assert np.all(np.abs(V[flips]) <= bound[flips])


def test_unfused_similarity_matches_oracle(hdc):
    cfg = CONFIGS["cfg1"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    Bd, Cd = to_dev(B, C)
    m = hdc.Model(Bd, Cd, prec="fp32_tc")
    H = m.encode(torch.from_numpy(X).cuda())
    y, S = hdc.similarity_packed(H, cfg.D, Cd)
    y_fused, S_fused = m.infer(torch.from_numpy(X).cuda(), return_scores=True)
    torch.cuda.synchronize()
    m.close()
    orc = oracle.infer(X, B, C, allow=True)
    rep = check_fp32(orc, y.cpu().numpy(), S.cpu().numpy())
    print("unfused", rep)
    assert np.array_equal(y.cpu().numpy(), y_fused.cpu().numpy())


def test_bundle_matches_oracle_exactly(hdc):
    rng = np.random.default_rng(2)
    N, F, D, K = 777, 61, 1000, 7
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    y = rng.integers(0, K, N).astype(np.int32)
    m = hdc.Model(torch.from_numpy(B).cuda(), None, prec="fp32_tc", K=K)
    H = m.encode(torch.from_numpy(X).cuda())
    counts, M = hdc.bundle_classes(H, D, torch.from_numpy(y).cuda(), K)
    torch.cuda.synchronize()
    m.close()
    c_o, M_o = oracle.train(oracle.encode(X, B), y, K)
    assert np.array_equal(counts.cpu().numpy().astype(np.int64), c_o)
    assert np.array_equal(M.cpu().numpy().astype(np.float64), M_o)


def test_bundle_accumulates_and_rejects_bad_labels(hdc):
    rng = np.random.default_rng(8)
    N, D, K = 100, 70, 3
    Hs = np.where(rng.random((N, D)) < 0.5, -1, 1).astype(np.int8)
    bits = (Hs < 0).astype(np.uint64)
    words = np.zeros((N, 3), dtype=np.uint32)
    for d in range(D):
        words[:, d // 32] |= (bits[:, d] << np.uint64(d % 32)).astype(np.uint32)
    H = torch.from_numpy(words.view(np.int32)).cuda()
    y = rng.integers(0, K, N).astype(np.int32)
    counts, _ = hdc.bundle_classes(H, D, torch.from_numpy(y).cuda(), K, return_M=False)
    counts, _ = hdc.bundle_classes(H, D, torch.from_numpy(y).cuda(), K, counts=counts, return_M=False)
    c_o, _ = oracle.train(Hs, y, K)
    assert np.array_equal(counts.cpu().numpy().astype(np.int64), 2 * c_o)
    bad = torch.from_numpy(np.array([0, 3] + [0] * (N - 2), dtype=np.int32)).cuda()
    with pytest.raises(hdc.HDCError):
        hdc.bundle_classes(H, D, bad, K)


def test_train_single_pass_end_to_end(hdc):
    # S:437 setting on the GPU: train, then infer with the trained class HVs
    rng = np.random.default_rng(0)
    F, D, K = 16, 2048, 3
    dirs = rng.standard_normal((K, F))
    centers = 3.0 * dirs / np.linalg.norm(dirs, axis=1, keepdims=True)
    y = rng.integers(0, K, 400).astype(np.int32)
    X = (centers[y] + rng.standard_normal((400, F))).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    Xd, Bd = to_dev(X, B)
    M, counts = hdc.train_single_pass(Xd[:200], torch.from_numpy(y[:200]).cuda(), Bd, K)
    c_o, M_o = oracle.train(oracle.encode(X[:200], B), y[:200], K)
    assert np.array_equal(M.cpu().numpy().astype(np.float64), M_o)
    m = hdc.Model(Bd, M, prec="fp32_tc")
    pred, _ = m.infer(Xd[200:])
    torch.cuda.synchronize()
    m.close()
    acc = float(np.mean(pred.cpu().numpy() == y[200:]))
    print("single-pass accuracy", acc)
    assert acc >= 0.95


def test_encode_full_size_cfg2_rows(hdc):
    # full cfg2 shape in the launch configuration inference uses; sampled rows vs oracle
    cfg = CONFIGS["cfg2"]
    X, B = make_X(cfg), make_B(cfg)
    m = hdc.Model(torch.from_numpy(B).cuda(), None, prec="fp32_tc", K=cfg.K)
    H = m.encode(torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    m.close()
    rows = np.r_[0:64, cfg.N - 64:cfg.N, np.random.default_rng(1).integers(0, cfg.N, 64)]
    Hg = _unpack(hdc, H[torch.from_numpy(rows).cuda()], cfg.D)
    assert np.array_equal(Hg, oracle.encode(X[rows], B))


def test_bundle_rejects_bad_labels_without_touching_counts(hdc):
    # validation happens on the device before any accumulation: on HDC_ERR_INVALID_VALUE the
    # caller's counts (and M) are exactly as they were
    rng = np.random.default_rng(5)
    N, D, K = 300, 700, 4
    H = torch.from_numpy(rng.integers(0, 2 ** 31, (N, (D + 31) // 32), dtype=np.int64).astype(np.int32)).cuda()
    y = torch.from_numpy(rng.integers(0, K, N).astype(np.int32)).cuda()
    y[17] = K                                              # out of range
    counts = torch.arange(K * D, dtype=torch.int32, device="cuda").reshape(K, D)
    before = counts.clone()
    with pytest.raises(hdc.HDCError):
        hdc.bundle_classes(H, D, y, K, counts=counts)
    torch.cuda.synchronize()
    assert torch.equal(counts, before)
    y[17] = -1
    with pytest.raises(hdc.HDCError):
        hdc.bundle_classes(H, D, y, K, counts=counts)
    assert torch.equal(counts, before)
