"""ctypes binding of the device generator twin (libhdcgen.so)."""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhdcgen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libhdcgen.so not built; run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        lib.hdcgen_uniform_f32.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_uint32, ctypes.c_uint32, ctypes.c_float,
                                           ctypes.c_float, ctypes.c_void_p]
        lib.hdcgen_uniform_f32.restype = ctypes.c_int
        _lib = lib
    return _lib


def uniform_f32_device(seed, tid, start, count, a, b, device, out=None):
    """Same bytes as hdc_inputs.philox.uniform_f32, generated on `device`."""
    if out is None:
        out = torch.empty(count, dtype=torch.float32, device=device)
    stream = torch.cuda.current_stream(device).cuda_stream
    rc = _load().hdcgen_uniform_f32(out.data_ptr(), start, count, seed, tid, a, b, stream)
    if rc:
        raise RuntimeError("hdcgen_uniform_f32 failed (%d)" % rc)
    return out


def make_X_device(cfg, device, r0=0, r1=None):
    r1 = cfg.N if r1 is None else r1
    x = uniform_f32_device(cfg.seed, 0, r0 * cfg.F, (r1 - r0) * cfg.F, cfg.x_lo, cfg.x_hi, device)
    return x.view(r1 - r0, cfg.F)
