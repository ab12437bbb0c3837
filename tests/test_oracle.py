"""Pins for the CPU oracle (oracle/): worked examples, brute force, invariants.

None of these re-derive the oracle's own formula: each compares against a value
fixed by the paper/SPEC, an exact-rational brute force, a library routine on a
special case, or a mathematical invariant."""
import json
import os

import numpy as np
import pytest

import oracle
from hdc_inputs import CONFIGS, make_B, make_C, make_X
from tests.bruteforce import exact_infer

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- worked examples
def test_hardsign_golden():
    g = _gold("hardsign.json")
    for case in g["cases"]:
        assert [oracle.hardsign(v) for v in case["v"]] == case["h"]
    assert oracle.hardsign(-0.0) == 1.0          # -0.0 >= 0 -> +1 (DESIGN R1)
    assert oracle.hardsign(-1e-300) == -1.0
    assert oracle.hardsign(5e-324) == 1.0


def test_encode_golden():
    for case in _gold("encode.json")["cases"]:
        X = np.array([case["x"]], dtype=np.float32)
        B = np.array(case["B"], dtype=np.float32)
        V = oracle.preact(X, B)
        assert V[0].tolist() == case["v"]
        D = B.shape[1]
        out = oracle.infer(X, B, np.eye(D, dtype=np.float32))   # C = I  ->  S = H
        assert out["S"][0].tolist() == case["h"]


def test_encode_basis_vector_selects_row():
    rng = np.random.default_rng(1)
    B = rng.standard_normal((5, 33)).astype(np.float32)
    for f in range(5):
        x = np.zeros((1, 5), np.float32)
        x[0, f] = 1.0
        out = oracle.infer(x, B, np.eye(33, dtype=np.float32))
        assert np.array_equal(out["S"][0], np.where(B[f] >= 0, 1.0, -1.0))


def test_similarity_golden():
    for case in _gold("similarity.json")["cases"]:
        h = np.array(case["h"], dtype=np.float32)
        X = np.ones((1, 1), np.float32)
        B = h[None, :]                        # F = 1, x = 1  ->  H = HardSign(h) = h
        C = np.array(case["C"], dtype=np.float32)
        out = oracle.infer(X, B, C)
        assert out["S"][0].tolist() == case["s"]


def test_argmax_golden():
    for case in _gold("argmax.json")["cases"]:
        C = np.array(case["s"], dtype=np.float32)[:, None]   # D = 1, H = [+1]  ->  S = C
        out = oracle.infer(np.ones((1, 1), np.float32), np.ones((1, 1), np.float32), C)
        assert int(out["y"][0]) == case["y"]


def test_zero_class_matrix_gives_zero_scores_label_zero():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((4, 6)).astype(np.float32)
    B = rng.standard_normal((6, 16)).astype(np.float32)
    out = oracle.infer(X, B, np.zeros((3, 16), np.float32))
    assert np.all(out["S"] == 0) and np.all(out["y"] == 0)      # S:107 + tie rule


def test_zero_row_encodes_all_plus_one():
    B = np.random.default_rng(3).standard_normal((7, 20)).astype(np.float32)
    X = np.zeros((2, 7), np.float32)
    X[1, :] = -0.0
    out = oracle.infer(X, B, np.eye(20, dtype=np.float32))
    assert np.all(out["S"] == 1.0)


def test_self_similarity_equals_D():
    rng = np.random.default_rng(4)
    D = 50
    h = np.where(rng.standard_normal(D) >= 0, 1.0, -1.0).astype(np.float32)
    C = np.stack([h, -h, np.ones(D, np.float32)])
    out = oracle.infer(np.ones((1, 1), np.float32), h[None, :], C)
    assert out["S"][0, 0] == D and out["y"][0] == 0


def test_duplicate_winning_classes_pick_lowest_index():
    rng = np.random.default_rng(5)
    X = rng.standard_normal((8, 5)).astype(np.float32)
    B = rng.standard_normal((5, 40)).astype(np.float32)
    base = rng.standard_normal((1, 40)).astype(np.float32)
    C = np.concatenate([-np.abs(base), base, base, base], axis=0)
    out = oracle.infer(X, B, C)
    # classes 1..3 are identical; whenever they win, label must be 1
    wins = out["S"][:, 1] >= out["S"][:, 0]
    assert np.all(out["y"][wins] == 1)


# ---------------------------------------------------------------- brute force
def _small_int_case(rng, force_zero=False):
    N, F, D, K = (int(rng.integers(1, 9)) for _ in range(4))
    X = rng.integers(-3, 4, size=(N, F)).astype(np.float32)
    B = rng.integers(-3, 4, size=(F, D)).astype(np.float32)
    C = rng.integers(-3, 4, size=(K, D)).astype(np.float32)
    if force_zero:
        X[0, :] = 0
        if K >= 2:
            C[K - 1] = C[0]                                     # force a tie candidate
    return X, B, C


@pytest.mark.parametrize("trial", range(60))
def test_bruteforce_small_integers_bitwise(trial):
    rng = np.random.default_rng(1000 + trial)
    X, B, C = _small_int_case(rng, force_zero=(trial % 3 == 0))
    V, H, S, y = exact_infer(X.tolist(), B.tolist(), C.tolist())
    out = oracle.infer(X, B, C)
    assert np.array_equal(out["S"], np.array([[float(s) for s in row] for row in S]))
    assert out["y"].tolist() == y
    Vo = oracle.preact(X, B)
    assert np.array_equal(Vo, np.array([[float(v) for v in row] for row in V]))


@pytest.mark.parametrize("trial", range(20))
def test_bruteforce_random_floats_within_rounding(trial):
    """Random fp32 data: the oracle's float64 sums stay within their rounding bound
    of the exact rational result, and every sign outside the ambiguity set agrees."""
    rng = np.random.default_rng(2000 + trial)
    N, F, D, K = (int(rng.integers(1, 9)) for _ in range(4))
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    V, H, S, y = exact_infer(X.tolist(), B.tolist(), C.tolist())
    Vo = oracle.preact(X, B)
    W = np.abs(X.astype(np.float64)) @ np.abs(B.astype(np.float64))
    Vx = np.array([[float(v) for v in row] for row in V])
    assert np.all(np.abs(Vo - Vx) <= (F + 1) * 2.0 ** -53 * W)
    out = oracle.infer(X, B, C)
    c1 = np.abs(C.astype(np.float64)).sum(axis=1)
    Sx = np.array([[float(s) for s in row] for row in S])
    assert np.all(np.abs(out["S"] - Sx) <= (D + 1) * 2.0 ** -53 * c1[None, :])


# ---------------------------------------------------------------- invariants
def test_linearity_exact_on_integers():
    rng = np.random.default_rng(7)
    X1 = rng.integers(-4, 5, (6, 9)).astype(np.float32)
    X2 = rng.integers(-4, 5, (6, 9)).astype(np.float32)
    B = rng.integers(-4, 5, (9, 30)).astype(np.float32)
    a, b = 3.0, -2.0
    V = oracle.preact(a * X1 + b * X2, B)
    assert np.array_equal(V, a * oracle.preact(X1, B) + b * oracle.preact(X2, B))


def test_linearity_random():
    rng = np.random.default_rng(8)
    X1 = rng.uniform(-1, 1, (5, 40)).astype(np.float32)
    X2 = rng.uniform(-1, 1, (5, 40)).astype(np.float32)
    B = rng.standard_normal((40, 64)).astype(np.float32)
    a, b = np.float32(0.75), np.float32(-1.5)                # exact fp32 scalings
    Xc = (a * X1 + b * X2).astype(np.float32)
    Xc64 = a * X1.astype(np.float64) + b * X2.astype(np.float64)
    exact_ok = np.array_equal(Xc.astype(np.float64), Xc64)
    V = oracle.preact(Xc, B)
    W = (np.abs(X1) * abs(a) + np.abs(X2) * abs(b)).astype(np.float64) @ np.abs(B.astype(np.float64))
    ref = float(a) * oracle.preact(X1, B) + float(b) * oracle.preact(X2, B)
    tol = 1e-12 * W if exact_ok else 1e-6 * W
    assert np.all(np.abs(V - ref) <= tol)


def _dchunk_scores(X, B, C, cuts):
    tot = None
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        part = oracle.infer(X, B[:, lo:hi], C[:, lo:hi])["S"]
        tot = part if tot is None else tot + part
    return tot


def test_dchunk_sum_exact_on_integers():
    """Alg. 3 `S += S_local`: summing partial scores over a D-partition
    equals the unchunked scores."""
    rng = np.random.default_rng(9)
    X = rng.integers(-3, 4, (7, 11)).astype(np.float32)
    B = rng.integers(-3, 4, (11, 97)).astype(np.float32)
    C = rng.integers(-3, 4, (5, 97)).astype(np.float32)
    full = oracle.infer(X, B, C)["S"]
    assert np.array_equal(_dchunk_scores(X, B, C, [0, 13, 14, 60, 97]), full)


def test_dchunk_sum_random():
    rng = np.random.default_rng(10)
    X = rng.uniform(-1, 1, (9, 31)).astype(np.float32)
    B = rng.standard_normal((31, 500)).astype(np.float32)
    C = rng.standard_normal((6, 500)).astype(np.float32)
    out = oracle.infer(X, B, C)
    part = _dchunk_scores(X, B, C, [0, 128, 256, 300, 499, 500])
    assert np.all(np.abs(part - out["S"]) <= 1e-12 * out["c1"][None, :])


def test_matches_library_matmul_special_case():
    """V equals numpy's float64 GEMM (a textbook routine, different summation
    order) within the float64 rounding bound."""
    rng = np.random.default_rng(11)
    X = rng.uniform(-1, 1, (12, 70)).astype(np.float32)
    B = rng.standard_normal((70, 130)).astype(np.float32)
    V = oracle.preact(X, B)
    ref = X.astype(np.float64) @ B.astype(np.float64)
    W = np.abs(X.astype(np.float64)) @ np.abs(B.astype(np.float64))
    assert np.all(np.abs(V - ref) <= 2 * 71 * 2.0 ** -53 * W)


def test_batch_structure_invariants():
    rng = np.random.default_rng(12)
    X = rng.uniform(-1, 1, (10, 13)).astype(np.float32)
    B = rng.standard_normal((13, 77)).astype(np.float32)
    C = rng.standard_normal((4, 77)).astype(np.float32)
    out = oracle.infer(X, B, C)
    # N = 1 equals the single-sample case; identical rows -> identical outputs
    for n in (0, 5, 9):
        one = oracle.infer(X[n:n + 1], B, C)
        assert np.array_equal(one["S"][0], out["S"][n]) and one["y"][0] == out["y"][n]
    X2 = np.concatenate([X[3:4], X[3:4]])
    dup = oracle.infer(X2, B, C)
    assert np.array_equal(dup["S"][0], dup["S"][1])
    # row permutation permutes outputs
    p = rng.permutation(10)
    perm = oracle.infer(X[p], B, C)
    assert np.array_equal(perm["S"], out["S"][p]) and np.array_equal(perm["y"], out["y"][p])
    # permuting K permutes S columns
    q = np.array([2, 0, 3, 1])
    pk = oracle.infer(X, B, C[q])
    assert np.array_equal(pk["S"], out["S"][:, q])
    # permuting D (columns of B and C) leaves S unchanged up to summation order
    r = rng.permutation(77)
    pd = oracle.infer(X, B[:, r], C[:, r])
    assert np.all(np.abs(pd["S"] - out["S"]) <= 1e-12 * out["c1"][None, :])


def test_dpermutation_exact_on_integers():
    rng = np.random.default_rng(13)
    X = rng.integers(-3, 4, (6, 8)).astype(np.float32)
    B = rng.integers(-3, 4, (8, 40)).astype(np.float32)
    C = rng.integers(-3, 4, (3, 40)).astype(np.float32)
    r = rng.permutation(40)
    assert np.array_equal(oracle.infer(X, B, C)["S"], oracle.infer(X, B[:, r], C[:, r])["S"])


def test_scaling_and_sign_metamorphic():
    rng = np.random.default_rng(14)
    X = rng.uniform(-1, 1, (8, 21)).astype(np.float32)
    B = rng.standard_normal((21, 90)).astype(np.float32)
    C = rng.standard_normal((5, 90)).astype(np.float32)
    out = oracle.infer(X, B, C)
    for k in (-3, 5):
        s = np.float32(2.0 ** k)
        o2 = oracle.infer(X * s, B, C)                    # H unchanged
        assert np.array_equal(o2["S"], out["S"]) and np.array_equal(o2["y"], out["y"])
        o3 = oracle.infer(X, B * s, C)
        assert np.array_equal(o3["S"], out["S"])
        o4 = oracle.infer(X, B, C * s)                    # S scales exactly
        assert np.array_equal(o4["S"], out["S"] * float(s)) and np.array_equal(o4["y"], out["y"])
    V = oracle.preact(X, B)
    assert np.array_equal(oracle.preact(-X, B), -V)       # RNE is sign-symmetric
    if not np.any(V == 0):
        assert np.array_equal(oracle.infer(-X, B, C)["S"], -out["S"])


def test_rejects_nonfinite_and_mismatch():
    X = np.ones((2, 3), np.float32)
    B = np.ones((3, 4), np.float32)
    C = np.ones((2, 4), np.float32)
    for bad in (np.nan, np.inf, -np.inf):
        Xb = X.copy()
        Xb[1, 2] = bad
        with pytest.raises(oracle.OracleError):
            oracle.infer(Xb, B, C)
        Cb = C.copy()
        Cb[0, 0] = bad
        with pytest.raises(oracle.OracleError):
            oracle.infer(X, B, Cb)
    with pytest.raises(oracle.OracleError):
        oracle.infer(X, np.ones((4, 4), np.float32), C)


def test_ambiguity_allowance_marks_exact_cancellations():
    # x = [1, 1], b_d = [1, -1] -> V = 0 with W = 2 > 0: ambiguous; zero rows are not.
    X = np.array([[1.0, 1.0], [0.0, 0.0]], np.float32)
    B = np.array([[1.0, 2.0], [-1.0, 1.0]], np.float32)
    C = np.array([[0.5, -1.0], [2.0, 3.0]], np.float32)
    out = oracle.infer(X, B, C, allow=True)
    assert out["namb"].tolist() == [1, 0]
    assert out["allow"][0].tolist() == [1.0, 4.0] and out["allow"][1].tolist() == [0.0, 0.0]


def test_threads_do_not_change_results():
    cfg = CONFIGS["cfg1"]
    X = make_X(cfg, 0, 16)
    B, C = make_B(cfg), make_C(cfg)
    a = oracle.infer(X, B, C, nthreads=1)
    b = oracle.infer(X, B, C, nthreads=4)
    assert np.array_equal(a["S"], b["S"]) and np.array_equal(a["y"], b["y"])


def test_generator_closed_forms_on_cfg1_sample():
    """||C_k||_1 ~ sqrt(2D/pi) for row-normalised Gaussian rows; mean |S| ~ 0.8
    (SURVEY §8c 'Generator sanity')."""
    cfg = CONFIGS["cfg1"]
    B, C = make_B(cfg), make_C(cfg)
    out = oracle.infer(make_X(cfg, 0, 32), B, C)
    assert np.all(np.abs(out["c1"] - np.sqrt(2 * cfg.D / np.pi)) < 1.5)
    assert 0.5 < np.mean(np.abs(out["S"])) < 1.1
