"""Property pins for the bf16 hi-plane sign bound of the small-batch kernel (DESIGN.md §4,
k_smallstream.cu hi_bound_kernel / HALF).

The kernel evaluates v_hi = fl32(x . b_hi) with b_hi = RN_bf16(b) and treats the sign as
decided unless |v_hi| <= ||x||_fp32 * beta_d + 1e-37, where

    beta_d = (||b_lo,d|| + tau_F ||b_hi,d||) (1 + 2 F u + 2^-10),  b_lo = b - b_hi (exact),
    tau_F = (F + 32) u (1 + 2 F u + 2^-16),  u = 2^-24 (common.cuh sign_bound_coef).

Claims checked here in plain numpy on the host (no GPU): (1) b_lo is exact in fp32 and
|b_lo| <= 2^-8 |b| (bf16 keeps 8 significant bits); (2) |x.b - v_hi| <= ||x|| beta_d for fp32 accumulation in two different
orders, on random and on cancellation-heavy data, so an unflagged v_hi has the exact sign;
(3) the flag rate at the cfg3 distribution is the few percent DESIGN.md states."""
import numpy as np
import pytest

U = 2.0 ** -24


def bf16_rn(a):
    """Round-to-nearest-even fp32 -> bf16 (returned as fp32), the kernel's __float2bfloat16_rn."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def tau_coef(F):
    return np.float32((F + 32) * U * (1.0 + 2.0 * F * U + 1.0 / 65536.0))


def beta(B):
    """Per-column bound coefficient (hi_bound_kernel), float64 then rounded up to fp32."""
    F = B.shape[0]
    hi = bf16_rn(B).astype(np.float64)
    lo = B.astype(np.float64) - hi
    b = (np.sqrt((lo * lo).sum(0)) + float(tau_coef(F)) * np.sqrt((hi * hi).sum(0))) * \
        (1.0 + 2.0 * F * U + 1.0 / 1024.0)
    b32 = b.astype(np.float32)
    return np.where(b32.astype(np.float64) < b, np.nextafter(b32, np.float32(np.inf)), b32)


def fl32_dot(x, bh, order):
    """fp32 fused multiply-add accumulation of x . b_hi (per column) in a given f order."""
    acc = np.zeros(bh.shape[1], dtype=np.float32)
    for f in order:
        # fmaf: one rounding of x*b + acc (the product of an fp32 and a bf16 is exact in fp64)
        acc = (np.float64(x[f]) * bh[f].astype(np.float64) + acc.astype(np.float64)).astype(np.float32)
    return acc


def test_residual_exact_and_small():
    rng = np.random.default_rng(0)
    b = np.concatenate([rng.standard_normal(20000), rng.uniform(-1e30, 1e30, 100),
                        rng.uniform(-1e-30, 1e-30, 100)]).astype(np.float32)
    hi = bf16_rn(b)
    lo32 = (b - hi).astype(np.float32)                      # fp32 subtraction
    lo64 = b.astype(np.float64) - hi.astype(np.float64)
    assert np.array_equal(lo32.astype(np.float64), lo64)   # exact in fp32
    nz = b != 0
    assert np.all(np.abs(lo64[nz]) <= 2.0 ** -8 * np.abs(b[nz].astype(np.float64)))


@pytest.mark.parametrize("kind", ["cfg3", "signed", "cancel"])
def test_unflagged_signs_are_exact(kind):
    rng = np.random.default_rng({"cfg3": 1, "signed": 2, "cancel": 3}[kind])
    F, D = 784, 600
    if kind == "cfg3":
        x = rng.uniform(0, 1, F).astype(np.float32)
        B = rng.standard_normal((F, D)).astype(np.float32)
    elif kind == "signed":
        x = rng.uniform(-1, 1, F).astype(np.float32)
        B = (rng.standard_normal((F, D)) * np.exp(rng.uniform(-8, 8, (F, 1)))).astype(np.float32)
    else:
        # last feature cancels the rest for every column: |v| tiny next to ||x|| ||b||
        x = rng.uniform(-1, 1, F).astype(np.float32)
        x[-1] = 1.0
        B = rng.standard_normal((F, D)).astype(np.float32)
        part = x[:-1].astype(np.float64) @ B[:-1].astype(np.float64)
        B[-1] = (-part + rng.uniform(-1e-2, 1e-2, D)).astype(np.float32)
    bh = bf16_rn(B)
    exact = x.astype(np.float64) @ B.astype(np.float64)    # products exact; fp64 sum error ~1e-16 W
    xnorm = np.float32(np.sqrt(np.float32((x.astype(np.float32) ** 2).sum(dtype=np.float32))))
    tau = xnorm.astype(np.float64) * beta(B).astype(np.float64) + 1e-37
    W = np.abs(x.astype(np.float64)) @ np.abs(B.astype(np.float64))
    for order in (np.arange(F), rng.permutation(F)):
        v = fl32_dot(x, bh, order).astype(np.float64)
        err = np.abs(v - exact)
        assert np.all(err <= tau - 1e-12 * W)              # the bound holds with room
        unflagged = np.abs(v) > tau
        assert np.all((v[unflagged] >= 0) == (exact[unflagged] >= 0))
    if kind == "cancel":
        assert np.mean(np.abs(v) <= tau) > 0.5              # the hard case is mostly flagged


def test_flag_rate_at_cfg3():
    rng = np.random.default_rng(4)
    F, D, N = 784, 2000, 8
    X = rng.uniform(0, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    bt = beta(B).astype(np.float64)
    V = X.astype(np.float64) @ bf16_rn(B).astype(np.float64)
    xn = np.sqrt((X.astype(np.float64) ** 2).sum(1))
    rate = np.mean(np.abs(V) <= xn[:, None] * bt[None, :])
    assert 0.01 < rate < 0.06                              # ~3% of elements
