"""Pins for the oracle's encoding and single-pass training (oracle.encode / oracle.train).

Single-pass training: class HVs by constrained bundling of the encoded
HVs of each class -- bundling is element-wise addition, normalised by HardSign
(ties +1).  Pinned against SPEC worked examples, an
exact-rational brute force, and invariants, never by retyping the formula."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests.bruteforce import exact_infer

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_bundling_golden():
    g = json.load(open(os.path.join(GOLD, "bundling.json")))
    for case in g["bundle_cases"]:
        H = np.array([case["h1"], case["h2"]], dtype=np.int8)
        counts, M = oracle.train(H, [0, 0], 1)
        assert counts[0].tolist() == case["sum"]
        assert M[0].tolist() == case["hardsign"]


def test_self_bundle_is_2h():
    # S:62 h (+) h -> 2h
    rng = np.random.default_rng(1)
    h = np.where(rng.random(37) < 0.5, -1, 1).astype(np.int8)
    counts, M = oracle.train(np.stack([h, h]), [0, 0], 1)
    assert np.array_equal(counts[0], 2 * h.astype(np.int64))
    assert np.array_equal(M[0], h.astype(np.float64))


def test_encode_matches_exact_rational():
    rng = np.random.default_rng(7)
    for trial in range(20):
        N, F, D = rng.integers(1, 5), rng.integers(1, 6), rng.integers(1, 7)
        X = rng.integers(-3, 4, (N, F)).astype(np.float32)
        B = rng.integers(-3, 4, (F, D)).astype(np.float32)
        if trial % 3 == 0:
            X[0] = 0.0                                   # zero row -> all +1
        _, Hx, _, _ = exact_infer(X.tolist(), B.tolist(), [[0.0] * int(D)])
        assert np.array_equal(oracle.encode(X, B), np.array(Hx, dtype=np.int8))


def test_train_matches_exact_rational_per_class():
    rng = np.random.default_rng(11)
    for _ in range(15):
        N, F, D, K = rng.integers(1, 9), rng.integers(1, 5), rng.integers(1, 9), rng.integers(1, 5)
        X = rng.integers(-3, 4, (N, F)).astype(np.float32)
        B = rng.integers(-3, 4, (F, D)).astype(np.float32)
        y = rng.integers(0, K, N).astype(np.int32)
        _, Hx, _, _ = exact_infer(X.tolist(), B.tolist(), [[0.0] * int(D)])
        cnt = [[Fraction(0)] * int(D) for _ in range(K)]
        for n in range(N):
            for d in range(D):
                cnt[y[n]][d] += Hx[n][d]
        counts, M = oracle.train(oracle.encode(X, B), y, K)
        assert counts.tolist() == [[int(c) for c in row] for row in cnt]
        assert M.tolist() == [[1.0 if c >= 0 else -1.0 for c in row] for row in cnt]


def test_singleton_class_is_the_encoded_sample():
    # one sample per class -> m_k = encode of that sample exactly
    rng = np.random.default_rng(3)
    X = rng.uniform(-1, 1, (4, 12)).astype(np.float32)
    B = rng.standard_normal((12, 300)).astype(np.float32)
    H = oracle.encode(X, B)
    _, M = oracle.train(H, np.arange(4), 4)
    assert np.array_equal(M, H.astype(np.float64))


def test_duplicated_set_gives_same_model():
    # duplicating the training set scales counts by 2, HardSign unchanged
    rng = np.random.default_rng(5)
    H = np.where(rng.random((30, 101)) < 0.5, -1, 1).astype(np.int8)
    y = rng.integers(0, 3, 30).astype(np.int32)
    c1, M1 = oracle.train(H, y, 3)
    c2, M2 = oracle.train(np.concatenate([H, H]), np.concatenate([y, y]), 3)
    assert np.array_equal(c2, 2 * c1)
    assert np.array_equal(M1, M2)


def test_permutation_and_total_invariants():
    # order of samples is irrelevant; sum over classes = sum over samples;
    # |count| <= n_k and count = n_k (mod 2)
    rng = np.random.default_rng(9)
    H = np.where(rng.random((64, 77)) < 0.5, -1, 1).astype(np.int8)
    y = rng.integers(0, 5, 64).astype(np.int32)
    c, M = oracle.train(H, y, 5)
    perm = rng.permutation(64)
    cp, Mp = oracle.train(H[perm], y[perm], 5)
    assert np.array_equal(c, cp) and np.array_equal(M, Mp)
    assert np.array_equal(c.sum(axis=0), H.astype(np.int64).sum(axis=0))
    nk = np.bincount(y, minlength=5)[:, None]
    assert np.all(np.abs(c) <= nk) and np.all((c - nk) % 2 == 0)


def test_label_out_of_range_rejected():
    with pytest.raises(oracle.OracleError):
        oracle.train(np.ones((2, 3), dtype=np.int8), [0, 2], 2)


def test_synthetic_clusters_accuracy():
    # S:437 (derived): 3 Gaussian clusters, F=16, 200 train / 200 test, D=2048 -> the
    # single-pass model classifies the held-out half with accuracy >= 0.95.  Reading of
    # "separation 3 sigma" (R13): class centres at distance 3 sigma from the
    # origin along random directions (HardSign(x B) encodes direction: no bias term).
    rng = np.random.default_rng(0)
    F, D, K = 16, 2048, 3
    dirs = rng.standard_normal((K, F))
    centers = 3.0 * dirs / np.linalg.norm(dirs, axis=1, keepdims=True)
    y = rng.integers(0, K, 400).astype(np.int32)
    X = (centers[y] + rng.standard_normal((400, F))).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    H = oracle.encode(X[:200], B)
    _, M = oracle.train(H, y[:200], K)
    out = oracle.infer(X[200:], B, M.astype(np.float32))
    assert np.mean(out["y"] == y[200:]) >= 0.95
