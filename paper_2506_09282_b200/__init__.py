"""B200-native batched HDC inference (ScalableHD, arXiv 2506.09282, hot path).

Public API: ``Model`` (resident B, C), ``infer`` (one-shot), ``argmax``, and the
sharding helpers in ``sharding``.  The compute runs in libhdc.so (sm_100a).
"""
from .hdc import HDCError, Model, PATH, PREC, argmax, infer, lib, LIB_PATH

__all__ = ["HDCError", "Model", "PATH", "PREC", "argmax", "infer", "lib", "LIB_PATH"]
