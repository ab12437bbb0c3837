"""Pins of the oracle's low-precision views (DESIGN.md §3 T1-T3, readings R15/R16):
operand rounding to tf32 / bf16, the oracle on rounded operands, and the rigorous
ambiguity allowances.  The TF32/BF16 paths are not in the paper (fp32 only, P:143,
P:538); these views only make the BASELINE north_star's TF32/BF16 tolerance precise."""
import numpy as np
import pytest
import torch

import oracle
from oracle.policy import check_lowp, check_rounded


def test_bf16_rounding_equals_torch_bfloat16():
    # library routine: torch's fp32 -> bfloat16 conversion (round to nearest even)
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(200000), rng.uniform(-1, 1, 50000) * 1e-30,
                        rng.uniform(-1, 1, 50000) * 1e30]).astype(np.float32)
    # exact halfway cases: a bf16 value plus half its ulp (ties -> even)
    base = torch.from_numpy(rng.standard_normal(1000).astype(np.float32)).bfloat16().float().numpy()
    half = np.ldexp(np.float32(1.0), np.frexp(base)[1] - 9).astype(np.float32)
    x = np.concatenate([x, base + half, base - half]).astype(np.float32)
    ref = torch.from_numpy(x).bfloat16().float().numpy()
    assert np.array_equal(oracle.round_fmt(x, "bf16"), ref)


def test_tf32_rounding_ties_away_hand_values():
    u = 2.0 ** -10                                  # tf32 ulp at 1
    cases = [(1 + u / 2, 1 + u),                    # tie -> away (even would give 1)
             (-(1 + u / 2), -(1 + u)),
             (1 + 2.5 * u, 1 + 3 * u),              # tie -> away (even would give 1 + 2u)
             (1 + u / 2 - 2.0 ** -20, 1.0),         # below the tie -> down
             (1 + 0.75 * u, 1 + u),
             (3.0, 3.0), (0.0, 0.0), (-0.0, -0.0),
             (2.0 ** 100 * (1 + u / 2), 2.0 ** 100 * (1 + u)),
             (0.1, 0.0999755859375)]                # 0.1 -> 1638 * 2^-14
    x = np.array([a for a, _ in cases], np.float32)
    r = oracle.round_fmt(x, "tf32")
    assert r.tolist() == [np.float32(b) for _, b in cases]
    assert np.signbit(r[7])                         # -0.0 stays -0.0


def test_rounding_keeps_representable_values_and_is_idempotent():
    rng = np.random.default_rng(1)
    ints = rng.integers(-255, 256, 10000).astype(np.float32)      # 8 significant bits
    assert np.array_equal(oracle.round_fmt(ints, "bf16"), ints)
    assert np.array_equal(oracle.round_fmt(ints, "tf32"), ints)
    x = rng.standard_normal(10000).astype(np.float32)
    for fmt in ("bf16", "tf32"):
        r = oracle.round_fmt(x, fmt)
        assert np.array_equal(oracle.round_fmt(r, fmt), r)
        u = oracle.UNIT_ROUNDOFF[fmt]
        assert np.all(np.abs(r.astype(np.float64) - x) <= u * np.abs(x.astype(np.float64)))


def test_rounded_oracle_equals_oracle_on_pre_rounded_operands():
    rng = np.random.default_rng(2)
    X = rng.uniform(-1, 1, (9, 30)).astype(np.float32)
    B = rng.standard_normal((30, 200)).astype(np.float32)
    C = rng.standard_normal((5, 200)).astype(np.float32)
    a = oracle.infer(X, B, C, fmt="bf16")
    Xr = torch.from_numpy(X).bfloat16().float().numpy()
    Br = torch.from_numpy(B).bfloat16().float().numpy()
    b = oracle.infer(Xr, Br, C)
    assert np.array_equal(a["S"], b["S"]) and np.array_equal(a["y"], b["y"])
    # small-integer operands are exact in every format: the same answer as fp32
    Xi = rng.integers(-3, 4, (9, 30)).astype(np.float32)
    Bi = rng.integers(-3, 4, (30, 200)).astype(np.float32)
    for fmt in ("tf32", "bf16"):
        assert np.array_equal(oracle.infer(Xi, Bi, C, fmt=fmt)["S"], oracle.infer(Xi, Bi, C)["S"])


def test_lowp_ambiguity_set_hand_case():
    # V = [2^-7, 2^-3, 0], W = [2 - 2^-7, 2 - 2^-3, 2]
    X = np.array([[1.0, 1.0]], np.float32)
    B = np.array([[1.0, 1.0, 1.0], [-1 + 2.0 ** -7, -1 + 2.0 ** -3, -1.0]], np.float32)
    C = np.array([[0.5, -7.0, 3.0], [-2.0, 11.0, 0.25]], np.float32)
    # bf16 (u = 2^-8): |V| <= ~(2^-7)W catches d = 0 and d = 2; tf32 (u = 2^-11): d = 2 only
    bf = oracle.infer(X, B, C, allow=True, gamma=oracle.gamma_lowp(2, "bf16"))
    assert bf["namb"].tolist() == [2]
    assert bf["allow"][0].tolist() == [2 * (0.5 + 3.0), 2 * (2.0 + 0.25)]
    tf = oracle.infer(X, B, C, allow=True, gamma=oracle.gamma_lowp(2, "tf32"))
    assert tf["namb"].tolist() == [1]
    assert tf["allow"][0].tolist() == [6.0, 0.5]


def test_accumulation_ambiguity_hand_case():
    # gamma_tc_acc(F=2) = 3 * 2^-22 ~ 7.2e-7: V = 2^-21 (W ~ 2) is inside, V = 2^-19 is not
    X = np.array([[1.0, 1.0]], np.float32)
    B = np.array([[1.0, 1.0], [-1 + 2.0 ** -21, -1 + 2.0 ** -19]], np.float32)
    C = np.array([[1.0, 10.0]], np.float32)
    o = oracle.infer(X, B, C, allow=True, gamma=oracle.gamma_tc_acc(2))
    assert o["namb"].tolist() == [1] and o["allow"][0].tolist() == [2.0]


@pytest.mark.parametrize("fmt", ["bf16", "tf32"])
def test_simulated_tensor_core_result_is_accepted(fmt):
    # an independent model of the TF32 / BF16 kernel: rounded operands (torch / oracle),
    # fp32 products summed by numpy's float32 GEMM (its own order), HardSign, fp64 Stage II.
    # Both views must accept it; the exact fp32 answer must be rejected by the rounded view
    # whenever the rounding moved a sign outside the accumulation set.
    rng = np.random.default_rng(3 if fmt == "bf16" else 4)
    N, F, D, K = 64, 200, 3000, 10
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    C /= np.linalg.norm(C.astype(np.float64), axis=1, keepdims=True).astype(np.float32)
    Xr, Br = oracle.round_fmt(X, fmt), oracle.round_fmt(B, fmt)
    V32 = Xr @ Br                                               # float32 accumulation
    H = np.where(V32 >= 0, 1.0, -1.0)
    S = H @ C.astype(np.float64).T
    y = np.argmax(S, axis=1).astype(np.int32)
    exact, rounded = oracle.infer_lowp(X, B, C, fmt)
    rep = check_lowp(exact, y, S, rtol=1e-2, rounded=rounded)
    assert rep["vs_rounded"]["score_violations"] == 0
    # the unrounded (exact) answer: where rounding moved a sign outside the accumulation
    # set, the rounded view must reject it (bf16 moves many such signs)
    V, Vr = oracle.preact(X, B), oracle.preact(Xr, Br)
    Wr = np.abs(Xr).astype(np.float64) @ np.abs(Br).astype(np.float64)
    outside = ((V >= 0) != (Vr >= 0)) & (np.abs(Vr) > oracle.gamma_tc_acc(F) * Wr)
    if fmt == "bf16":
        assert outside.sum() > 100
    Sx = np.where(V >= 0, 1.0, -1.0) @ C.astype(np.float64).T
    if outside.any():
        with pytest.raises(AssertionError):
            check_rounded(rounded, np.argmax(Sx, 1).astype(np.int32), Sx)
