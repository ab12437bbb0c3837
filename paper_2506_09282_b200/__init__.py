"""B200-native batched HDC inference (ScalableHD, arXiv 2506.09282, hot path).

Public API: ``Model`` (resident B, C; ``encode`` for Stage I alone), ``infer``
(one-shot), ``argmax``, the materialised-H helpers ``similarity_packed`` (unfused
ablation), ``bundle_classes`` / ``train_single_pass`` (single-pass training),
and the sharding helpers in ``sharding``.  The compute runs in libhdc.so (sm_100a).
"""
from .hdc import (HDCError, LIB_PATH, Model, PATH, PREC, argmax, bundle_classes, diag_stream_read,
                  dshard_exchange_bytes, infer, lib, similarity_packed, train_single_pass, unpack_signs)

__all__ = ["HDCError", "Model", "PATH", "PREC", "argmax", "infer", "lib", "LIB_PATH",
           "similarity_packed", "bundle_classes", "train_single_pass", "unpack_signs", "dshard_exchange_bytes",
           "diag_stream_read"]
