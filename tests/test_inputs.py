"""Seeded input generator (hdc_inputs): known answers, exactness, row-range
consistency, distribution sanity; the device twin equals the host bit for bit."""
import numpy as np
import pytest

from hdc_inputs import CONFIGS, make_B, make_C, make_X
from hdc_inputs.philox import philox4x32_10, uniform_f32, uniform_u32, normal_f64


def test_philox_known_answers():
    # Random123 philox4x32_10 known-answer vectors
    out = philox4x32_10(0, 0, 0, 0, 0, 0)
    assert [int(v) for v in out] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    m = 0xFFFFFFFF
    out = philox4x32_10(m, m, m, m, m, m)
    assert [int(v) for v in out] == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    out = philox4x32_10(0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0)
    assert [int(v) for v in out] == [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_uniform_ranges_exact():
    u = uniform_f32(0, 0, 0, 100000, -1.0, 1.0)
    assert u.dtype == np.float32 and u.min() >= -1.0 and u.max() < 1.0
    # every value is k * 2^-23 exactly
    k = u.astype(np.float64) * 2.0 ** 23
    assert np.array_equal(k, np.round(k))
    v = uniform_f32(0, 0, 0, 100000, 0.0, 1.0)
    assert v.min() >= 0.0 and v.max() < 1.0
    assert abs(v.mean() - 0.5) < 0.01 and abs(u.mean()) < 0.01


def test_subranges_consistent():
    full = uniform_u32(7, 3, 0, 1001)
    for s, c in [(0, 1), (1, 5), (3, 9), (998, 3), (517, 100)]:
        assert np.array_equal(uniform_u32(7, 3, s, c), full[s:s + c])
    nf = normal_f64(7, 3, 0, 103)
    assert np.array_equal(normal_f64(7, 3, 5, 50), nf[5:55])
    cfg = CONFIGS["cfg1"]
    X = make_X(cfg)
    assert np.array_equal(make_X(cfg, 17, 40), X[17:40])


def test_streams_differ():
    a = uniform_u32(0, 0, 0, 64)
    assert not np.array_equal(a, uniform_u32(0, 1, 0, 64))
    assert not np.array_equal(a, uniform_u32(1, 0, 0, 64))


def test_normal_statistics():
    z = normal_f64(0, 1, 0, 400000)
    assert abs(z.mean()) < 4 / np.sqrt(z.size)
    assert abs(z.var() - 1.0) < 0.01
    assert abs(np.mean(np.abs(z)) - np.sqrt(2 / np.pi)) < 0.005


def test_config_tensors():
    cfg = CONFIGS["cfg1"]
    B, C = make_B(cfg), make_C(cfg)
    assert B.shape == (561, 10000) and B.dtype == np.float32
    assert C.shape == (6, 10000)
    assert np.allclose(np.linalg.norm(C.astype(np.float64), axis=1), 1.0, atol=1e-6)
    X = make_X(CONFIGS["cfg3_n4"])
    assert X.shape == (4, 784) and X.min() >= 0


@pytest.mark.gpu
def test_device_generator_matches_host(cuda_device):
    from hdc_inputs.device import uniform_f32_device
    for (s, c, a, b) in [(0, 1, -1.0, 1.0), (3, 1001, -1.0, 1.0), (617 * 5, 617 * 33, 0.0, 1.0)]:
        dev = uniform_f32_device(0, 0, s, c, a, b, cuda_device).cpu().numpy()
        assert np.array_equal(dev, uniform_f32(0, 0, s, c, a, b))
