"""BASELINE.json configs as seeded synthetic inputs.

Stand-ins for the paper's datasets (ISOLET F=617 K=26, SA12 F=561,
MNIST F=784 K=10, D=10000) and its TrainableHD-trained B and M, which
are not available: X ~ U[-1,1) (cfg1, cfg2) or U[0,1) (cfg3-5), B ~ N(0,1),
C ~ N(0,1) with rows L2-normalised (normalised in float64, rounded to fp32).
Seed 0; Philox streams X=0, B=1, C=2.
"""
import hashlib
from dataclasses import dataclass

import numpy as np

from .philox import uniform_f32, normal_f64

TID_X, TID_B, TID_C = 0, 1, 2


@dataclass(frozen=True)
class Config:
    name: str
    N: int
    F: int
    D: int
    K: int
    x_lo: float
    x_hi: float
    seed: int = 0


CONFIGS = {
    "cfg1": Config("cfg1", 256, 561, 10000, 6, -1.0, 1.0),
    "cfg2": Config("cfg2", 16384, 617, 10000, 26, -1.0, 1.0),
    "cfg3_n1": Config("cfg3_n1", 1, 784, 10000, 10, 0.0, 1.0),
    "cfg3_n4": Config("cfg3_n4", 4, 784, 10000, 10, 0.0, 1.0),
    "cfg3_n16": Config("cfg3_n16", 16, 784, 10000, 10, 0.0, 1.0),
    "cfg3_n32": Config("cfg3_n32", 32, 784, 10000, 10, 0.0, 1.0),
    "cfg4": Config("cfg4", 262144, 784, 10000, 10, 0.0, 1.0),
    "cfg5": Config("cfg5", 131072, 3072, 10000, 10, 0.0, 1.0),
    "cfg5_d2000": Config("cfg5_d2000", 131072, 3072, 2000, 10, 0.0, 1.0),
    "cfg5_d20000": Config("cfg5_d20000", 131072, 3072, 20000, 10, 0.0, 1.0),
}


def make_X(cfg, r0=0, r1=None):
    """Rows [r0, r1) of X (N x F fp32, row-major). Element (n, f) has index n*F+f."""
    r1 = cfg.N if r1 is None else r1
    x = uniform_f32(cfg.seed, TID_X, r0 * cfg.F, (r1 - r0) * cfg.F, cfg.x_lo, cfg.x_hi)
    return x.reshape(r1 - r0, cfg.F)


def make_B(cfg):
    """B (F x D fp32): i.i.d. N(0,1) (P:119 'sampled from a Gaussian distribution')."""
    return normal_f64(cfg.seed, TID_B, 0, cfg.F * cfg.D).astype(np.float32).reshape(cfg.F, cfg.D)


def make_C(cfg):
    """C (K x D fp32): N(0,1), each row divided by its L2 norm in float64, then rounded."""
    z = normal_f64(cfg.seed, TID_C, 0, cfg.K * cfg.D).reshape(cfg.K, cfg.D)
    z = z / np.sqrt(np.sum(z * z, axis=1, keepdims=True))
    return z.astype(np.float32)


def tensor_hash(a):
    """Digest of an array's bytes (provenance for result rows)."""
    return hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=8).hexdigest()
