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
        lib.oracle_infer_ex.argtypes = [P, P, P, I64, I64, I64, I64, ctypes.c_int, ctypes.c_double,
                                        P, P, P, P, ctypes.c_int]
        lib.oracle_infer_ex.restype = ctypes.c_int
        lib.oracle_round_array.argtypes = [P, I64, ctypes.c_int, P]
        lib.oracle_round_array.restype = ctypes.c_int
        lib.oracle_round_fmt.argtypes = [ctypes.c_double, ctypes.c_int]
        lib.oracle_round_fmt.restype = ctypes.c_double
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


FMT = {"fp32": 0, "tf32": 1, "bf16": 2}
# unit roundoff of the operand formats (round to nearest, p explicit mantissa bits: 2^-(p+1))
UNIT_ROUNDOFF = {"fp32": 2.0 ** -24, "tf32": 2.0 ** -11, "bf16": 2.0 ** -8}


def round_fmt(a, fmt):
    """Round every element of an fp32 array to tf32 (nearest, ties away) or bf16
    (nearest, ties even), returned as fp32 (oracle_round_fmt, R15)."""
    a = _f32(a)
    out = np.empty_like(a)
    rc = _load().oracle_round_array(_ptr(a), a.size, FMT[fmt], _ptr(out))
    if rc:
        raise OracleError("bad format")
    return out


def gamma_fp64(F):
    """A64: float64 summation of F exact products, |fl(V) - V| <= (F-1) 2^-53 W < (F+1) 2^-53 W."""
    return (F + 1) * 2.0 ** -53


def gamma_tc_acc(F, u=0.0):
    """Tensor-core fp32 accumulation of F products (derivation T1): each
    product enters the sum with at most one fp32 ulp of alignment truncation and one of
    accumulator rounding, 2 * 2^-23 relative to sum |terms|; terms of operands rounded
    with unit roundoff u are bounded by (1+u)^2 |x b|."""
    return (F + 1) * 2.0 ** -22 * (1.0 + u) ** 2


def gamma_lowp(F, fmt):
    """Rigorous TF32 / BF16 ambiguity (T2): |fl(x) fl(b) - x b| <= (2u + u^2)|x b|
    plus the tensor-core accumulation bound, so every d with |V| > gamma W keeps its sign."""
    u = UNIT_ROUNDOFF[fmt]
    return 2 * u + u * u + gamma_tc_acc(F, u) + gamma_fp64(F)


def infer(X, B, C, allow=False, nthreads=1, fmt="fp32", gamma=None):
    """Alg. 1: returns dict with S (float64 N x K), y (int32 N),
    and, if ``allow``, the allowance (N x K) over the ambiguity set
    {d : W > 0, |V| <= gamma W} (default gamma: A64, float64 rounding) and the
    ambiguous counts (N).  ``fmt`` = "tf32" / "bf16" rounds X and B to that
    operand format before Stage I (R15).  Also margin (top-2 gap),
    rowscale max_k |S|, and c1 = ||C_k||_1."""
    X, B, C = _f32(X), _f32(B), _f32(C)
    if X.ndim != 2 or B.ndim != 2 or C.ndim != 2:
        raise OracleError("expected 2-D X, B, C")
    N, F = X.shape
    F2, D = B.shape
    K, D2 = C.shape
    if F != F2 or D != D2:
        raise OracleError("dimension mismatch")
    if gamma is None:
        gamma = gamma_fp64(F)
    S = np.empty((N, K), dtype=np.float64)
    y = np.empty(N, dtype=np.int32)
    al = np.empty((N, K), dtype=np.float64) if allow else None
    na = np.empty(N, dtype=np.int32) if allow else None
    rc = _load().oracle_infer_ex(_ptr(X), _ptr(B), _ptr(C), N, F, D, K, FMT[fmt], float(gamma),
                                 _ptr(S), _ptr(y), _ptr(al) if allow else None,
                                 _ptr(na) if allow else None, int(nthreads))
    if rc:
        raise OracleError("non-finite input" if rc == 1 else "oracle error %d" % rc)
    out = {"S": S, "y": y, "allow": al, "namb": na, "gamma": float(gamma), "fmt": fmt}
    if K >= 2:
        srt = np.sort(S, axis=1)
        out["margin"] = srt[:, -1] - srt[:, -2]
    else:
        out["margin"] = np.full(N, np.inf)
    out["rowscale"] = np.max(np.abs(S), axis=1) if N else np.zeros(0)
    out["c1"] = np.sum(np.abs(C.astype(np.float64)), axis=1)
    out["D"] = D
    return out


def infer_lowp(X, B, C, fmt, nthreads=1):
    """The two oracle views a TF32 / BF16 result is judged against:
    "exact": the exact problem with the rigorous low-precision ambiguity allowance
    (gamma_lowp), and "rounded": the problem on operands rounded to ``fmt`` with the
    tensor-core accumulation allowance (gamma_tc_acc)."""
    F = np.shape(X)[1]
    exact = infer(X, B, C, allow=True, nthreads=nthreads, gamma=gamma_lowp(F, fmt))
    rounded = infer(X, B, C, allow=True, nthreads=nthreads, fmt=fmt, gamma=gamma_tc_acc(F))
    return exact, rounded


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
