"""Negative pins of the comparison policy (oracle/policy.py): every check must REJECT a
result that is wrong by more than the tolerance BASELINE north_star states (fp32 path:
1e-4 relative on scores, identical labels outside near-ties; TF32/BF16: 1e-2 relative,
disagreements only at near-ties), and accept the oracle's own answer.  Readings R10/R11
(DESIGN.md §3): "relative" is relative to ||C_k||_1; |S| in the margin rule is max_k |S|."""
import numpy as np
import pytest

import oracle
from oracle.policy import check_fp32, check_lowp, check_rounded, self_consistent, stage2_rel


def _problem(N=64, F=40, D=900, K=6, seed=5):
    rng = np.random.default_rng(seed)
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    C /= np.linalg.norm(C.astype(np.float64), axis=1, keepdims=True).astype(np.float32)
    return X, B, C


@pytest.fixture(scope="module")
def fp32_case():
    X, B, C = _problem()
    orc = oracle.infer(X, B, C, allow=True)
    return orc


def _clear_margin_row(orc, rtol):
    """A row whose top-2 margin is well outside twice the tolerance rtol * max c1."""
    ok = orc["margin"] > 2.5 * rtol * orc["c1"].max()
    return int(np.nonzero(ok)[0][0])


def test_fp32_accepts_the_oracle_itself(fp32_case):
    orc = fp32_case
    rep = check_fp32(orc, orc["y"], orc["S"].astype(np.float32))
    assert rep["label_mismatch"] == 0 and rep["score_violations"] == 0


def test_fp32_rejects_score_off_by_2e_4_c1(fp32_case):
    orc = fp32_case
    S = orc["S"].copy()
    S[3, 2] += 2e-4 * orc["c1"][2]              # twice the 1e-4 tolerance on one element
    y = np.argmax(S, axis=1).astype(np.int32)
    with pytest.raises(AssertionError, match="score tolerance"):
        check_fp32(orc, y, S)
    S[3, 2] -= 1.5e-4 * orc["c1"][2]            # 0.5e-4: inside, accepted
    check_fp32(orc, np.argmax(S, axis=1).astype(np.int32), S)


def test_fp32_rejects_swapped_label_outside_near_tie(fp32_case):
    orc = fp32_case
    n = _clear_margin_row(orc, 1e-4)
    y = orc["y"].copy()
    y[n] = (y[n] + 1) % orc["S"].shape[1]
    with pytest.raises(AssertionError, match="label mismatch"):
        check_fp32(orc, y)                                  # labels only
    with pytest.raises(AssertionError):
        check_fp32(orc, y, orc["S"])                        # not the argmax of these scores


def test_fp32_accepts_a_near_tie_swap_only():
    # two classes with equal scores up to < 1e-4 * max|S|: either label is acceptable,
    # a label whose score is further below is not
    orc = {"S": np.array([[1.0, 1.0 - 1e-6, 0.2]]), "y": np.array([0], np.int32),
           "allow": np.zeros((1, 3)), "c1": np.array([50.0, 50.0, 50.0]),
           "margin": np.array([1e-6]), "rowscale": np.array([1.0])}
    rep = check_fp32(orc, np.array([1]))
    assert rep["exempt_rows"] == 1 and rep["label_mismatch"] == 1
    with pytest.raises(AssertionError, match="near-tie"):
        check_fp32(orc, np.array([2]))


def test_fp32_rejects_out_of_range_and_inconsistent_labels(fp32_case):
    orc = fp32_case
    y = orc["y"].copy()
    y[0] = orc["S"].shape[1]
    with pytest.raises(AssertionError, match="out of range"):
        check_fp32(orc, y)
    y = orc["y"].copy()
    y[0] = -1
    with pytest.raises(AssertionError, match="out of range"):
        check_fp32(orc, y)
    S = orc["S"].copy()
    assert not self_consistent(S, (orc["y"] + 1) % S.shape[1])
    # ties: the lowest index is the only self-consistent label
    assert self_consistent(np.array([[2.0, 2.0]]), np.array([0]))
    assert not self_consistent(np.array([[2.0, 2.0]]), np.array([1]))


def test_fp32_allowance_widens_exactly_where_the_oracle_says():
    # exact cancellation: V[0, 0] = 0 (ambiguous in float64 terms), flipping h moves S by 2|C|
    X = np.array([[1.0, 1.0]], np.float32)
    B = np.array([[1.0, 1.0], [-1.0, 2.0]], np.float32)
    C = np.array([[0.5, 3.0], [2.0, -1.0]], np.float32)
    orc = oracle.infer(X, B, C, allow=True)
    assert orc["allow"][0].tolist() == [1.0, 4.0]
    S_flip = orc["S"].copy()
    S_flip[0] -= 2 * C[:, 0]                                # h_0 = -1 instead of +1
    check_fp32(orc, np.argmax(S_flip, 1).astype(np.int32), S_flip)
    S_bad = orc["S"].copy()
    S_bad[0] -= 2 * C[:, 1]                                 # a flip of the non-ambiguous column:
    assert abs(S_bad[0, 0] - orc["S"][0, 0]) > orc["allow"][0, 0] + 1e-4 * orc["c1"][0]  # 6 > 1
    with pytest.raises(AssertionError):
        check_fp32(orc, np.argmax(S_bad, 1).astype(np.int32), S_bad)


@pytest.fixture(scope="module")
def lowp_case():
    X, B, C = _problem(N=96, F=64, D=4000, K=8, seed=9)
    exact, rounded = oracle.infer_lowp(X, B, C, "bf16")
    return X, B, C, exact, rounded


def test_lowp_accepts_the_rounded_oracle(lowp_case):
    # the exact method on bf16-rounded operands is a valid bf16 answer under both checks
    X, B, C, exact, rounded = lowp_case
    S = rounded["S"]
    rep = check_lowp(exact, rounded["y"], S, rounded=rounded)
    assert rep["vs_rounded"]["score_violations"] == 0
    assert 0.0 < rep["amb_per_row"] < 4000


def test_lowp_rejects_score_off_by_1_1e_2_c1(lowp_case):
    X, B, C, exact, rounded = lowp_case
    S = exact["S"].copy()
    S[7, 3] += 1.1e-2 * exact["c1"][3]
    with pytest.raises(AssertionError, match="score tolerance"):
        check_lowp(exact, np.argmax(S, 1).astype(np.int32), S, rtol=1e-2)


def test_lowp_rejects_error_beyond_the_rigorous_allowance(lowp_case):
    # without north_star's 1e-2 (edge shapes), the rigorous allowance still binds
    X, B, C, exact, rounded = lowp_case
    n, k = 11, 5
    tol = exact["allow"][n, k] + stage2_rel(exact["D"]) * exact["c1"][k]
    S = exact["S"].copy()
    S[n, k] += 1.01 * tol
    with pytest.raises(AssertionError, match="score tolerance"):
        check_lowp(exact, np.argmax(S, 1).astype(np.int32), S, rtol=None)
    S[n, k] -= 0.02 * tol
    check_lowp(exact, np.argmax(S, 1).astype(np.int32), S, rtol=None)


def test_lowp_rejects_clear_label_disagreement(lowp_case):
    X, B, C, exact, rounded = lowp_case
    n = _clear_margin_row(exact, 1e-2)
    y = exact["y"].copy()
    y[n] = int(np.argmin(exact["S"][n]))
    with pytest.raises(AssertionError, match="label disagreement"):
        check_lowp(exact, y, rtol=1e-2)


def test_rounded_check_rejects_one_sign_flip_outside_its_set(lowp_case):
    # the rounded-operand check is ~100x tighter: one flipped sign outside the
    # accumulation-ambiguity set (|V_r| > gamma W_r) is rejected
    X, B, C, exact, rounded = lowp_case
    Xr, Br = oracle.round_fmt(X, "bf16"), oracle.round_fmt(B, "bf16")
    V = oracle.preact(Xr, Br)
    W = np.abs(Xr).astype(np.float64) @ np.abs(Br).astype(np.float64)
    n = 4
    d = int(np.argmax(np.abs(V[n]) / W[n]))                 # the safest sign of the row
    S = rounded["S"].copy()
    S[n] -= 2 * np.sign(V[n, d]) * C[:, d]
    with pytest.raises(AssertionError, match="score tolerance"):
        check_rounded(rounded, np.argmax(S, 1).astype(np.int32), S)
    check_lowp(exact, np.argmax(S, 1).astype(np.int32), S)   # still a valid bf16 answer
