"""CPU oracle for batched HDC inference -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package. The
product path (``paper_2506_09282_b200``) never does; it shares no code with it.

The arithmetic lives in ``hdc_oracle.c`` (plain float64 loops, the definition of
Alg. 1). This wrapper only marshals numpy arrays and derives
summary statistics (margins, scales) from the oracle's scores.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hdc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force=False):
    """Compile hdc_oracle.c with gcc (-O2, OpenMP, no FP contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
                               "-ffp-contract=off", "-fno-fast-math", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        lib.oracle_preact.argtypes = [P, P, I64, I64, I64, P]
        lib.oracle_preact.restype = ctypes.c_int
        lib.oracle_infer.argtypes = [P, P, P, I64, I64, I64, I64, P, P, P, P, ctypes.c_int]
        lib.oracle_infer.restype = ctypes.c_int
        lib.oracle_hardsign.argtypes = [ctypes.c_double]
        lib.oracle_hardsign.restype = ctypes.c_double
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_encode.argtypes = [P, P, I64, I64, I64, P]
        lib.oracle_encode.restype = ctypes.c_int
        lib.oracle_train.argtypes = [P, P, I64, I64, I64, P, P]
        lib.oracle_train.restype = ctypes.c_int
        _lib = lib
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(ValueError):
    pass


def hardsign(x):
    """HardSign of one value (eq. hardsign)."""
    return _load().oracle_hardsign(float(x))


def hardsign_vec(v):
    return np.array([hardsign(x) for x in np.asarray(v, dtype=np.float64).ravel()]).reshape(np.shape(v))


def num_threads():
    return _load().oracle_num_threads()


def preact(X, B):
    """V = X B in float64 (eq. batch_encode before act)."""
    X, B = _f32(X), _f32(B)
    N, F = X.shape
    F2, D = B.shape
    if F != F2:
        raise OracleError("dimension mismatch")
    V = np.empty((N, D), dtype=np.float64)
    rc = _load().oracle_preact(_ptr(X), _ptr(B), N, F, D, _ptr(V))
    if rc:
        raise OracleError("non-finite input" if rc == 1 else "oracle error %d" % rc)
    return V


def infer(X, B, C, allow=False, nthreads=1):
    """Alg. 1: returns dict with S (float64 N x K), y (int32 N),
    and, if ``allow``, the A64 allowance (N x K) and ambiguous counts (N).
    Also margin (top-2 gap), rowscale max_k |S|, and c1 = ||C_k||_1."""
    X, B, C = _f32(X), _f32(B), _f32(C)
    if X.ndim != 2 or B.ndim != 2 or C.ndim != 2:
        raise OracleError("expected 2-D X, B, C")
    N, F = X.shape
    F2, D = B.shape
    K, D2 = C.shape
    if F != F2 or D != D2:
        raise OracleError("dimension mismatch")
    S = np.empty((N, K), dtype=np.float64)
    y = np.empty(N, dtype=np.int32)
    al = np.empty((N, K), dtype=np.float64) if allow else None
    na = np.empty(N, dtype=np.int32) if allow else None
    rc = _load().oracle_infer(_ptr(X), _ptr(B), _ptr(C), N, F, D, K, _ptr(S), _ptr(y),
                              _ptr(al) if allow else None, _ptr(na) if allow else None,
                              int(nthreads))
    if rc:
        raise OracleError("non-finite input" if rc == 1 else "oracle error %d" % rc)
    out = {"S": S, "y": y, "allow": al, "namb": na}
    if K >= 2:
        srt = np.sort(S, axis=1)
        out["margin"] = srt[:, -1] - srt[:, -2]
    else:
        out["margin"] = np.full(N, np.inf)
    out["rowscale"] = np.max(np.abs(S), axis=1) if N else np.zeros(0)
    out["c1"] = np.sum(np.abs(C.astype(np.float64)), axis=1)
    return out


def encode(X, B):
    """H = HardSign(X B) as int8 +-1 (eq. batch_encode, HardSign P:126-131)."""
    X, B = _f32(X), _f32(B)
    N, F = X.shape
    F2, D = B.shape
    if F != F2:
        raise OracleError("dimension mismatch")
    H = np.empty((N, D), dtype=np.int8)
    rc = _load().oracle_encode(_ptr(X), _ptr(B), N, F, D, _ptr(H))
    if rc:
        raise OracleError("non-finite input" if rc == 1 else "oracle error %d" % rc)
    return H


def train(H, y, K):
    """Single-pass training: counts[k] = sum of H rows of class k (int64),
    M = HardSign(counts) (float64 +-1, ties +1)."""
    H = np.ascontiguousarray(H, dtype=np.int8)
    y = np.ascontiguousarray(y, dtype=np.int32)
    N, D = H.shape
    counts = np.empty((K, D), dtype=np.int64)
    M = np.empty((K, D), dtype=np.float64)
    rc = _load().oracle_train(_ptr(H), _ptr(y), N, D, K, _ptr(counts), _ptr(M))
    if rc:
        raise OracleError("label outside [0, K)" if rc == 3 else "oracle error %d" % rc)
    return counts, M
