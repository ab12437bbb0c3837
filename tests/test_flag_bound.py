"""Property pins for the int8 epilogue's coarse flag test (k_fused_tc.cu phase 1).

The kernel never forms I = r0 2^14 + r1 2^7 + r2 (the exact int8-limb image of x.b) in 64 bits;
it tests J = (r0 << (14 - s)) + (r1 >> (s - 7)) + (r2 >> s) (arithmetic shifts, 7 <= s <= 14)
against the ceilings of the row and column taus over 2^s:

    flag  <=>  J' <= mrow + mcol,   J' = J if J >= 0 else -J - 1,
    mrow = ceil(tau_row / 2^s), mcol = ceil(tau_col / 2^s),

and takes the provisional sign from J.  The claims checked here with exact Python integers:
(1) every element with |I| <= tau_row + tau_col is flagged (the rigorous bound of DESIGN §4
is never weakened); (2) an unflagged element has sign(J) = sign(I); (3) J fits in 32 bits for
|r| within the limb ranges at F <= 100000 with s = tc_flag_shift(Fp)."""
import random

import pytest


def tc_flag_shift(Fp):
    """Mirror of k_fused_tc.cu tc_flag_shift (host arithmetic only)."""
    s = 0
    while (1 << (s + 1)) < Fp:
        s += 1
    return min(max(s, 7), 14)


def coarse(r0, r1, r2, s):
    return (r0 << (14 - s)) + (r1 >> (s - 7)) + (r2 >> s)   # Python >> is arithmetic (floor)


def ceil_div_pow2(t, s):
    return -((-t) >> s)


def flagged(r0, r1, r2, s, tau_row, tau_col):
    J = coarse(r0, r1, r2, s)
    Jp = J if J >= 0 else -J - 1
    return Jp <= ceil_div_pow2(tau_row, s) + ceil_div_pow2(tau_col, s), J


@pytest.mark.parametrize("Fp", [64, 128, 576, 640, 832, 3072, 8192, 32768, 100032])
def test_shift_range_and_32_bit_J(Fp):
    s = tc_flag_shift(Fp)
    assert 7 <= s <= 14
    # |r0| <= 2^14 Fp, |r1| <= 2^15 Fp, |r2| <= 3 2^14 Fp (three int8 limb products per element)
    J = coarse(2 ** 14 * Fp, 2 ** 15 * Fp, 3 * 2 ** 14 * Fp, s)
    Jn = coarse(-(2 ** 14) * Fp, -(2 ** 15) * Fp, -3 * 2 ** 14 * Fp, s)
    assert max(abs(J), abs(Jn) + 1) + 2 ** 28 < 2 ** 31      # J' - mcol with mcol >= -2^28


def _cases(rng, n, s):
    for _ in range(n):
        scale = rng.choice([1, 2 ** 6, 2 ** 12, 2 ** 20, 2 ** 30])
        r0 = rng.randint(-scale, scale)
        r1 = rng.randint(-scale, scale)
        r2 = rng.randint(-scale, scale)
        yield r0, r1, r2


@pytest.mark.parametrize("s", [7, 9, 11, 14])
def test_every_bound_element_is_flagged_and_signs_exact(s):
    rng = random.Random(1000 + s)
    for r0, r1, r2 in _cases(rng, 20000, s):
        I = r0 * 2 ** 14 + r1 * 2 ** 7 + r2
        # taus: positive (valid rows / columns), around |I| so that both sides of the bound occur
        base = abs(I) + rng.randint(-3 * 2 ** s, 3 * 2 ** s)
        tau_row = max(1, base // 2 + rng.randint(-5, 5))
        tau_col = max(1, base - tau_row + rng.randint(-5, 5))
        fl, J = flagged(r0, r1, r2, s, tau_row, tau_col)
        if abs(I) <= tau_row + tau_col:
            assert fl, (r0, r1, r2, s, tau_row, tau_col)
        if not fl:
            assert (J < 0) == (I < 0), (r0, r1, r2, s)
            assert I != 0


@pytest.mark.parametrize("s", [7, 10, 14])
def test_exact_boundary_cases(s):
    # I exactly at +-tau, one past it, zero and tiny negatives (floor shifts round towards -inf)
    for I in [0, -1, 1, -(2 ** s), 2 ** s, -(2 ** s) - 1, 5 * 2 ** s + 3, -(5 * 2 ** s) - 3]:
        for r1 in (-64, 0, 63):
            for r2 in (-64, 0, 63):
                rest = I - r1 * 2 ** 7 - r2
                if rest % 2 ** 14:
                    continue
                r0 = rest // 2 ** 14
                for tau in (abs(I), abs(I) + 1, max(abs(I) - 1, 1), 1):
                    tr = tau // 2 + 1
                    tc = max(tau - tr, 1)
                    fl, J = flagged(r0, r1, r2, s, tr, tc)
                    if abs(I) <= tr + tc:
                        assert fl
                    if not fl:
                        assert (J < 0) == (I < 0)


def test_padding_sentinels_never_flag():
    # rows past N (mrow = -2^28) and columns past D (mcol = -2^28): never flagged
    s = 10
    for J in (0, 1, -1, 2 ** 29, -(2 ** 29)):
        Jp = J if J >= 0 else -J - 1
        assert not (Jp - (-(2 ** 28)) <= 300)        # column past D, any valid row
        assert not (Jp - 300 <= -(2 ** 28))          # row past N, any valid column
