"""Thin Python binding of libhdc.so (include/hdc.h) over torch CUDA tensors.

Argument marshalling only: every step of the hot path runs in the library's
kernels.  There is no fallback: if libhdc.so is missing or a call fails, this
module raises.
"""
import ctypes
import os

import torch

LIB_PATH = os.environ.get("HDC_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "libhdc.so")

PREC = {"fp32": 0, "tf32": 1, "bf16": 2, "fp32_tc": 3}
PATH = {"auto": 0, "small": 1, "fused": 2}
KERNELS = {0: "none", 1: "small", 2: "ffma", 3: "tc", 4: "small_tc"}
_STATUS = {0: "HDC_OK", 1: "HDC_ERR_INVALID_VALUE", 2: "HDC_ERR_MISALIGNED",
           3: "HDC_ERR_UNSUPPORTED", 4: "HDC_ERR_NO_MEMORY", 5: "HDC_ERR_CUDA"}

_lib = None


class HDCError(RuntimeError):
    def __init__(self, status, detail):
        super().__init__("%s: %s" % (_STATUS.get(status, status), detail))
        self.status = status


def lib():
    """Load libhdc.so (raises if it has not been built -- no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libhdc.so not found at %s; run __graft_entry__.build()" % LIB_PATH)
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.hdc_infer.argtypes = [P, P, P, I64, I64, I64, I64, P, P, I32, P]
        L.hdc_model_create.argtypes = [P, P, I64, I64, I64, I32, ctypes.POINTER(P)]
        L.hdc_model_infer.argtypes = [P, P, I64, P, P, P]
        L.hdc_model_infer_path.argtypes = [P, P, I64, P, P, I32, P]
        L.hdc_model_infer_host.argtypes = [P, P, I64, P, P, P]
        L.hdc_model_partial_scores.argtypes = [P, P, I64, P, P]
        L.hdc_argmax.argtypes = [P, I64, I64, P, P]
        L.hdc_model_infer_dshard.argtypes = [P, P, I64, P, P, P, I32, I32, ctypes.c_uint32, P]
        L.hdc_dshard_exchange_bytes.argtypes = [I64, I64, I32]
        L.hdc_dshard_exchange_bytes.restype = I64
        L.hdc_model_encode.argtypes = [P, P, I64, P, I64, P]
        L.hdc_similarity_packed.argtypes = [P, I64, I64, I64, P, I64, P, P, P]
        L.hdc_bundle_classes.argtypes = [P, I64, I64, I64, P, I64, P, P, P]
        L.hdc_model_destroy.argtypes = [P]
        L.hdc_model_dims.argtypes = [P, P, P, P, P]
        L.hdc_model_recheck_count.argtypes = [P]
        L.hdc_model_recheck_count.restype = I64
        L.hdc_model_last_launch_count.argtypes = [P]
        L.hdc_model_last_launch_count.restype = ctypes.c_int32
        L.hdc_model_last_kernel.argtypes = [P]
        L.hdc_model_last_kernel.restype = ctypes.c_int32
        L.hdc_model_tc_tile_n.argtypes = [P]
        L.hdc_model_tc_tile_n.restype = ctypes.c_int32
        L.hdc_model_set_kernel_timing.argtypes = [P, I32]
        L.hdc_model_set_kernel_timing.restype = I32
        L.hdc_model_last_kernel_ms.argtypes = [P]
        L.hdc_model_last_kernel_ms.restype = ctypes.c_float
        L.hdc_status_string.argtypes = [I32]
        L.hdc_status_string.restype = ctypes.c_char_p
        L.hdc_last_error.restype = ctypes.c_char_p
        L.hdc_version.restype = ctypes.c_char_p
        L.hdc_diag_stream_read.argtypes = [P, I64, P]
        L.hdc_diag_stream_read.restype = I32
        for name in ("hdc_infer", "hdc_model_create", "hdc_model_infer", "hdc_model_infer_path",
                     "hdc_model_infer_host", "hdc_model_partial_scores", "hdc_argmax",
                     "hdc_model_infer_dshard",
                     "hdc_model_destroy", "hdc_model_dims", "hdc_model_encode",
                     "hdc_similarity_packed", "hdc_bundle_classes"):
            getattr(L, name).restype = I32
        _lib = L
    return _lib


def _check(status):
    if status != 0:
        raise HDCError(status, lib().hdc_last_error().decode())


def _stream_ptr(stream, device):
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _dev_f32(t, name):
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32):
        raise TypeError("%s must be a CUDA float32 tensor" % name)
    return t.contiguous()


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _rows(X, F, name="X"):
    """X must be a 2-D (N x F) CUDA float32 tensor; returns it contiguous."""
    X = _dev_f32(X, name)
    if X.dim() != 2 or X.shape[1] != F:
        raise ValueError("%s must be N x F = ? x %d, got %s" % (name, F, tuple(X.shape)))
    return X


def _out(t, dtype, numel, device, name):
    """A caller-supplied output: right dtype, contiguous, >= numel elements, on `device`
    (a torch.device: CUDA for the device entry points, CPU for the host one).  The C
    layer writes numel elements through the raw pointer, so a short or strided tensor
    would be overrun -- reject it instead."""
    if not isinstance(t, torch.Tensor):
        raise TypeError("%s must be a torch tensor" % name)
    if t.dtype != dtype:
        raise TypeError("%s must be %s, got %s" % (name, dtype, t.dtype))
    if not t.is_contiguous():
        raise ValueError("%s must be contiguous" % name)
    if t.numel() < numel:
        raise ValueError("%s has %d elements, needs %d" % (name, t.numel(), numel))
    if t.device.type != device.type or (device.type == "cuda" and t.device != device):
        raise ValueError("%s must be on %s, is on %s" % (name, device, t.device))
    return t


class Model:
    """A resident model (hdc_model_create): B (F x D) and C (K x D) on the device."""

    def __init__(self, B, C, prec="fp32", K=None):
        """C = None makes an encoder-only model (hdc_model_encode; K classes for training)."""
        B = _dev_f32(B, "B")
        if C is not None:
            C = _dev_f32(C, "C")
            if B.dim() != 2 or C.dim() != 2 or B.shape[1] != C.shape[1]:
                raise ValueError("B must be F x D and C K x D")
        elif B.dim() != 2:
            raise ValueError("B must be F x D")
        self.F, self.D = B.shape
        self.K = C.shape[0] if C is not None else int(K or 1)
        self.prec = prec
        self.device = B.device
        self._h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib().hdc_model_create(_ptr(B), _ptr(C), self.F, self.D, self.K, PREC[prec],
                                          ctypes.byref(self._h)))

    def infer(self, X, labels=None, scores=None, path="auto", stream=None, return_scores=False):
        """Labels (int32 N) and optionally scores (fp32 N x K) for X (N x F)."""
        X = _rows(X, self.F)
        N = X.shape[0]
        labels = self._labels(labels, N, X.device)
        scores = self._scores(scores, return_scores, N, X.device)
        with torch.cuda.device(self.device):
            _check(lib().hdc_model_infer_path(self._h, _ptr(X), N, _ptr(labels), _ptr(scores),
                                              PATH[path], _stream_ptr(stream, X.device)))
        return labels, scores

    def encode(self, X, H=None, stream=None):
        """Stage I only: bit-packed H (N x ceil(D/32) int32 words; bit set <=> h = -1)."""
        X = _rows(X, self.F)
        N = X.shape[0]
        ldw = (self.D + 31) // 32
        if H is None:
            H = torch.empty(N, ldw, dtype=torch.int32, device=X.device)
        elif H.dim() != 2 or H.shape[0] != N or H.shape[1] < ldw:
            raise ValueError("H must be N x (>= ceil(D/32)) int32 words")
        _out(H, torch.int32, N * ldw, X.device, "H")
        with torch.cuda.device(self.device):
            _check(lib().hdc_model_encode(self._h, _ptr(X), N, _ptr(H), H.shape[1],
                                          _stream_ptr(stream, X.device)))
        return H

    def infer_host(self, X_host, labels_host, scores_host=None, stream=None):
        """End-to-end call on (pinned) host tensors; asynchronous on `stream`."""
        if X_host.is_cuda or X_host.dtype != torch.float32 or not X_host.is_contiguous():
            raise TypeError("X_host must be a contiguous host float32 tensor")
        if X_host.dim() != 2 or X_host.shape[1] != self.F:
            raise ValueError("X_host must be N x F = ? x %d" % self.F)
        N = X_host.shape[0]
        cpu = torch.device("cpu")
        _out(labels_host, torch.int32, N, cpu, "labels_host")
        if scores_host is not None:
            _out(scores_host, torch.float32, N * self.K, cpu, "scores_host")
        with torch.cuda.device(self.device):
            _check(lib().hdc_model_infer_host(self._h, _ptr(X_host), N, _ptr(labels_host),
                                              _ptr(scores_host), _stream_ptr(stream, self.device)))
        return labels_host, scores_host

    def partial_scores(self, X, out=None, stream=None):
        """Scores over this model's D-slice, no argmax (D-shard piece, Alg. 3)."""
        X = _rows(X, self.F)
        N = X.shape[0]
        if out is None:
            out = torch.empty(N, self.K, dtype=torch.float32, device=X.device)
        _out(out, torch.float32, N * self.K, X.device, "out")
        with torch.cuda.device(self.device):
            _check(lib().hdc_model_partial_scores(self._h, _ptr(X), N, _ptr(out),
                                                  _stream_ptr(stream, X.device)))
        return out

    def infer_dshard(self, X, xbufs, rank, world, epoch, labels=None, scores=None, return_scores=False,
                     stream=None):
        """D-shard inference with the cross-rank sum inside the kernel
        (hdc_model_infer_dshard): `xbufs` is a CUDA int64 tensor of the `world` exchange
        buffer addresses (this rank's D-slice model; same X, N <= 32 and epoch on all ranks)."""
        X = _rows(X, self.F)
        if not (isinstance(xbufs, torch.Tensor) and xbufs.is_cuda and xbufs.dtype == torch.int64
                and xbufs.numel() == world and xbufs.is_contiguous()):
            raise TypeError("xbufs must be a contiguous CUDA int64 tensor of `world` addresses")
        N = X.shape[0]
        labels = self._labels(labels, N, X.device)
        scores = self._scores(scores, return_scores, N, X.device)
        with torch.cuda.device(self.device):
            _check(lib().hdc_model_infer_dshard(self._h, _ptr(X), N, _ptr(labels), _ptr(scores), _ptr(xbufs),
                                                int(rank), int(world), int(epoch) & 0xFFFFFFFF,
                                                _stream_ptr(stream, X.device)))
        return labels, scores

    def _labels(self, labels, N, device):
        if labels is None:
            return torch.empty(N, dtype=torch.int32, device=device)
        return _out(labels, torch.int32, N, device, "labels")

    def _scores(self, scores, want, N, device):
        if scores is None:
            return torch.empty(N, self.K, dtype=torch.float32, device=device) if want else None
        return _out(scores, torch.float32, N * self.K, device, "scores")

    def recheck_count(self):
        return int(lib().hdc_model_recheck_count(self._h))

    def last_launch_count(self):
        return int(lib().hdc_model_last_launch_count(self._h))

    def last_kernel(self):
        """Kernel family of the last call: "none", "small", "ffma" or "tc" (hdc_model_last_kernel)."""
        return KERNELS.get(int(lib().hdc_model_last_kernel(self._h)), "invalid")

    def tc_tile_n(self):
        """D-tile width of the fused tensor-core kernel (160: int8 wide mode), 0 if none."""
        return int(lib().hdc_model_tc_tile_n(self._h))

    def set_kernel_timing(self, enable=True):
        _check(lib().hdc_model_set_kernel_timing(self._h, 1 if enable else 0))

    def last_kernel_ms(self):
        return float(lib().hdc_model_last_kernel_ms(self._h))

    def close(self):
        if self._h:
            _check(lib().hdc_model_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def infer(X, B, C, prec="fp32", return_scores=False, stream=None):
    """One-shot hdc_infer(X, B, C, N, F, D, K) -> labels (+ scores)."""
    X, B, C = _dev_f32(X, "X"), _dev_f32(B, "B"), _dev_f32(C, "C")
    if X.dim() != 2 or B.dim() != 2 or C.dim() != 2 or X.shape[1] != B.shape[0] or C.shape[1] != B.shape[1]:
        raise ValueError("X (N x F), B (F x D), C (K x D) expected")
    if not (X.device == B.device == C.device):
        raise ValueError("X, B, C must be on one device")
    N, F = X.shape
    D = B.shape[1]
    K = C.shape[0]
    labels = torch.empty(N, dtype=torch.int32, device=X.device)
    scores = torch.empty(N, K, dtype=torch.float32, device=X.device) if return_scores else None
    with torch.cuda.device(X.device):
        _check(lib().hdc_infer(_ptr(X), _ptr(B), _ptr(C), N, F, D, K, _ptr(labels), _ptr(scores),
                               PREC[prec], _stream_ptr(stream, X.device)))
    return labels, scores


def diag_stream_read(buf, nbytes=None, stream=None):
    """One-shot bulk-copy read of a CUDA tensor's bytes (measurement diagnostic)."""
    if not (isinstance(buf, torch.Tensor) and buf.is_cuda and buf.is_contiguous()):
        raise TypeError("buf must be a contiguous CUDA tensor")
    n = buf.numel() * buf.element_size() if nbytes is None else int(nbytes)
    if n > buf.numel() * buf.element_size():
        raise ValueError("nbytes exceeds the buffer")
    with torch.cuda.device(buf.device):
        _check(lib().hdc_diag_stream_read(_ptr(buf), n, _stream_ptr(stream, buf.device)))


def dshard_exchange_bytes(N, K, world):
    """Bytes of one rank's exchange buffer for hdc_model_infer_dshard."""
    return int(lib().hdc_dshard_exchange_bytes(int(N), int(K), int(world)))


def argmax(S, labels=None, stream=None):
    """Lowest-index row argmax of S (N x K) -> int32 labels (hdc_argmax)."""
    S = _dev_f32(S, "S")
    if S.dim() != 2:
        raise ValueError("S must be N x K")
    N, K = S.shape
    if labels is None:
        labels = torch.empty(N, dtype=torch.int32, device=S.device)
    else:
        _out(labels, torch.int32, N, S.device, "labels")
    with torch.cuda.device(S.device):
        _check(lib().hdc_argmax(_ptr(S), N, K, _ptr(labels), _stream_ptr(stream, S.device)))
    return labels


def unpack_signs(H, D):
    """Packed H (N x ldw int32) -> N x D tensor of +-1 (test / inspection helper)."""
    bits = (H.view(torch.int32).unsqueeze(-1) >> torch.arange(32, device=H.device, dtype=torch.int32)) & 1
    bits = bits.reshape(H.shape[0], -1)[:, :D]
    return 1 - 2 * bits.to(torch.int8)


def _packed(H, D):
    if not (isinstance(H, torch.Tensor) and H.is_cuda and H.dtype == torch.int32 and H.dim() == 2
            and H.is_contiguous() and H.shape[1] >= (D + 31) // 32):
        raise TypeError("H must be a contiguous CUDA int32 tensor N x (>= ceil(D/32))")


def similarity_packed(H, D, C, labels=None, scores=None, return_scores=True, stream=None):
    """Stage II + argmax over a packed H (the unfused ablation path)."""
    C = _dev_f32(C, "C")
    _packed(H, D)
    N, ldw = H.shape
    K = C.shape[0]
    if C.dim() != 2 or C.shape[1] != D:
        raise ValueError("C must be K x D")
    if labels is None:
        labels = torch.empty(N, dtype=torch.int32, device=H.device)
    else:
        _out(labels, torch.int32, N, H.device, "labels")
    if scores is None and return_scores:
        scores = torch.empty(N, K, dtype=torch.float32, device=H.device)
    elif scores is not None:
        _out(scores, torch.float32, N * K, H.device, "scores")
    with torch.cuda.device(H.device):
        _check(lib().hdc_similarity_packed(_ptr(H), ldw, N, D, _ptr(C), K, _ptr(labels), _ptr(scores),
                                           _stream_ptr(stream, H.device)))
    return labels, scores


def bundle_classes(H, D, y, K, counts=None, return_M=True, stream=None):
    """Single-pass training: counts[k] += sum of h_n over class k; M = HardSign(counts)."""
    _packed(H, D)
    N, ldw = H.shape
    if not (isinstance(y, torch.Tensor) and y.device == H.device and y.numel() == N):
        raise ValueError("y must hold N labels on H's device")
    y = y.to(torch.int32).contiguous()
    if counts is None:
        counts = torch.zeros(K, D, dtype=torch.int32, device=H.device)
    else:
        _out(counts, torch.int32, K * D, H.device, "counts")
    M = torch.empty(K, D, dtype=torch.float32, device=H.device) if return_M else None
    with torch.cuda.device(H.device):
        _check(lib().hdc_bundle_classes(_ptr(H), ldw, N, D, _ptr(y), K, _ptr(counts), _ptr(M),
                                        _stream_ptr(stream, H.device)))
    return counts, M


def train_single_pass(X, y, B, K, prec="fp32_tc"):
    """Class HVs from labelled data: M = HardSign(sum over class of HardSign(x B))."""
    m = Model(B, None, prec=prec, K=K)
    try:
        H = m.encode(X)
        counts, M = bundle_classes(H, m.D, y, K)
    finally:
        m.close()
    return M, counts
