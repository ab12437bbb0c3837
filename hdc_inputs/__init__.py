"""Seeded synthetic input generator shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no encoding, no similarity, no
argmax). It only draws the inputs X, B, C of SURVEY.md §8d / BASELINE.json
configs with a counter-based generator (Philox4x32-10), so that:

* the host (numpy) path and the device path (``libhdcgen.so``) produce the same
  bytes for uniforms (pure integer arithmetic + one exact fp32 affine map);
* any row range of X can be regenerated independently (N-shards, row samples).

Normals (B and C) are drawn on the host only (Box-Muller in float64 uses
transcendental functions, whose last-ulp behaviour differs between libm and
CUDA), then copied to the device.
"""
from .philox import philox4x32_10, uniform_u32, uniform_f32, normal_f64, KEY_HI
from .configs import CONFIGS, Config, make_X, make_B, make_C, tensor_hash

__all__ = [
    "philox4x32_10", "uniform_u32", "uniform_f32", "normal_f64", "KEY_HI",
    "CONFIGS", "Config", "make_X", "make_B", "make_C", "tensor_hash",
]
