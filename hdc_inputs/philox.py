"""Philox4x32-10 counter-based generator (numpy, vectorised).

Stream layout (SURVEY.md §8c reading 12): key = (seed, KEY_HI); the 128-bit
counter of element ``idx`` of tensor ``tid`` is
``(idx >> 2 low 32, idx >> 2 high 32, tid, 0)`` and the element takes word
``idx & 3`` of the 4-word output block. The CUDA twin is
``hdc_inputs/csrc/hdcgen.cu``; both must stay bit-identical (tested).
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint32(0x9E3779B9)
W1 = np.uint32(0xBB67AE85)
KEY_HI = 0x48444331  # "HDC1": fixed high key word, the seed is the low word
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32 with 10 rounds. All inputs uint32 arrays/scalars."""
    c0 = np.asarray(c0, dtype=np.uint32)
    c1 = np.asarray(c1, dtype=np.uint32)
    c2 = np.asarray(c2, dtype=np.uint32)
    c3 = np.asarray(c3, dtype=np.uint32)
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    for r in range(10):
        if r > 0:
            k0 = np.uint32((int(k0) + int(W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(W1)) & 0xFFFFFFFF)
        p0 = M0 * c0.astype(np.uint64)
        p1 = M1 * c2.astype(np.uint64)
        hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
        lo0 = (p0 & _MASK).astype(np.uint32)
        hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
        lo1 = (p1 & _MASK).astype(np.uint32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def _blocks(start, count):
    """Counter blocks covering element indices [start, start+count)."""
    b0 = start >> 2
    b1 = (start + count + 3) >> 2
    blk = np.arange(b0, b1, dtype=np.uint64)
    return blk, int(start - (b0 << 2))


def uniform_u32(seed, tid, start, count):
    """Raw 32-bit words for element indices [start, start+count) of tensor tid."""
    if count == 0:
        return np.zeros(0, dtype=np.uint32)
    blk, off = _blocks(int(start), int(count))
    lo = (blk & _MASK).astype(np.uint32)
    hi = (blk >> np.uint64(32)).astype(np.uint32)
    w = philox4x32_10(lo, hi, np.uint32(tid), np.uint32(0), seed & 0xFFFFFFFF, KEY_HI)
    words = np.stack(w, axis=1).reshape(-1)
    return words[off:off + count]


def uniform_f32(seed, tid, start, count, a, b):
    """U[a, b) in fp32: u = (w >> 8) * 2^-24, x = a + (b - a) * u.

    For (a, b) in {(-1, 1), (0, 1)} every value is exact in fp32.
    """
    w = uniform_u32(seed, tid, start, count)
    u = (w >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
    return (np.float32(a) + np.float32(b - a) * u).astype(np.float32)


def normal_f64(seed, tid, start, count):
    """Standard normals in float64 by Box-Muller; 4 normals per Philox block.

    Word pair (w0, w1) -> (r cos t, r sin t), pair (w2, w3) likewise, with
    u1 = (w + 1) * 2^-32 in (0, 1] and t = 2*pi*w' * 2^-32.
    """
    if count == 0:
        return np.zeros(0, dtype=np.float64)
    blk, off = _blocks(int(start), int(count))
    lo = (blk & _MASK).astype(np.uint32)
    hi = (blk >> np.uint64(32)).astype(np.uint32)
    w0, w1, w2, w3 = philox4x32_10(lo, hi, np.uint32(tid), np.uint32(0),
                                   seed & 0xFFFFFFFF, KEY_HI)
    s = 2.0 ** -32
    r1 = np.sqrt(-2.0 * np.log((w0.astype(np.float64) + 1.0) * s))
    t1 = 2.0 * np.pi * (w1.astype(np.float64) * s)
    r2 = np.sqrt(-2.0 * np.log((w2.astype(np.float64) + 1.0) * s))
    t2 = 2.0 * np.pi * (w3.astype(np.float64) * s)
    z = np.stack([r1 * np.cos(t1), r1 * np.sin(t1), r2 * np.cos(t2), r2 * np.sin(t2)], axis=1)
    return z.reshape(-1)[off:off + count]
