"""Host-side checks of the C-ABI boundary (no GPU needed): the library loads,
exports every entry point include/hdc.h declares, and rejects bad arguments
synchronously without touching the device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2506_09282_b200 import build as b
    b.build()
    import paper_2506_09282_b200 as pkg
    return pkg.lib()


def _declared():
    src = open(os.path.join(ROOT, "include", "hdc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hdc_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for required in ("hdc_infer", "hdc_model_create", "hdc_model_infer", "hdc_model_partial_scores",
                     "hdc_argmax", "hdc_model_destroy", "hdc_status_string", "hdc_last_error"):
        assert required in names


def test_every_declared_symbol_is_exported(L):
    for name in _declared():
        assert hasattr(L, name), "libhdc.so does not export %s" % name


def test_status_strings(L):
    L.hdc_status_string.restype = ctypes.c_char_p
    assert L.hdc_status_string(0) == b"HDC_OK"
    assert L.hdc_status_string(1) == b"HDC_ERR_INVALID_VALUE"
    assert L.hdc_status_string(5) == b"HDC_ERR_CUDA"
    assert b"sm_100a" in L.hdc_version()


def test_invalid_arguments_rejected_synchronously(L):
    P = ctypes.c_void_p
    h = P()
    # F = 0
    assert L.hdc_model_create(P(16), P(16), 0, 10, 2, 0, ctypes.byref(h)) == 1
    # K > 256
    assert L.hdc_model_create(P(16), P(16), 4, 10, 257, 0, ctypes.byref(h)) == 1
    # null B
    assert L.hdc_model_create(None, P(16), 4, 10, 2, 0, ctypes.byref(h)) == 1
    # misaligned C
    assert L.hdc_model_create(P(16), P(18), 4, 10, 2, 0, ctypes.byref(h)) == 2
    # bad precision
    assert L.hdc_model_create(P(16), P(16), 4, 10, 2, 9, ctypes.byref(h)) == 1
    # F too large for the recheck bound
    assert L.hdc_model_create(P(16), P(16), (1 << 20) + 1, 10, 2, 0, ctypes.byref(h)) == 3
    assert b"F" in L.hdc_last_error()
    # argmax: negative N, K = 0, null pointers, misaligned
    assert L.hdc_argmax(P(16), -1, 3, P(16), None) == 1
    assert L.hdc_argmax(P(16), 4, 0, P(16), None) == 1
    assert L.hdc_argmax(None, 4, 3, P(16), None) == 1
    assert L.hdc_argmax(P(17), 4, 3, P(16), None) == 2
    # N = 0 is a no-op
    assert L.hdc_argmax(None, 0, 3, None, None) == 0
    # null model handle
    assert L.hdc_model_infer(None, P(16), 4, P(16), None, None) == 1
    assert L.hdc_model_destroy(None) == 1
    assert L.hdc_model_recheck_count(None) == -1


def test_binding_fails_loudly_without_cuda_tensors():
    import torch
    import paper_2506_09282_b200 as hdc
    with pytest.raises(TypeError):
        hdc.argmax(torch.zeros(3, 4))          # host tensor: no CPU fallback exists


def test_binding_rejects_mismatched_outputs_before_the_c_call():
    # the C layer writes N (N*K) elements through raw pointers: the binding must refuse
    # outputs of the wrong dtype, size, layout or device instead of letting it overrun
    import torch
    from paper_2506_09282_b200.hdc import _out
    cpu = torch.device("cpu")
    ok = torch.empty(8, dtype=torch.int32)
    assert _out(ok, torch.int32, 8, cpu, "labels") is ok
    with pytest.raises(TypeError):
        _out(torch.empty(8, dtype=torch.int64), torch.int32, 8, cpu, "labels")     # int64 labels
    with pytest.raises(ValueError):
        _out(torch.empty(7, dtype=torch.int32), torch.int32, 8, cpu, "labels")     # too short
    with pytest.raises(ValueError):
        _out(torch.empty(16, dtype=torch.int32)[::2], torch.int32, 8, cpu, "labels")  # strided
    with pytest.raises(ValueError):
        _out(ok, torch.int32, 8, torch.device("cuda", 0), "labels")               # wrong device
    with pytest.raises(TypeError):
        _out([0] * 8, torch.int32, 8, cpu, "labels")


@pytest.mark.gpu
def test_binding_rejects_wrong_widths_and_outputs_on_gpu(cuda_device):
    import torch
    import paper_2506_09282_b200 as hdc
    B = torch.randn(20, 300, device=cuda_device)
    C = torch.randn(4, 300, device=cuda_device)
    m = hdc.Model(B, C, prec="fp32_tc")
    X = torch.randn(10, 20, device=cuda_device)
    with pytest.raises(ValueError):
        m.infer(torch.randn(10, 19, device=cuda_device))
    with pytest.raises(ValueError):
        m.encode(torch.randn(10, 21, device=cuda_device))
    with pytest.raises(ValueError):
        m.partial_scores(torch.randn(10, 19, device=cuda_device))
    with pytest.raises(ValueError):
        m.infer(X, labels=torch.empty(9, dtype=torch.int32, device=cuda_device))
    with pytest.raises(TypeError):
        m.infer(X, labels=torch.empty(10, dtype=torch.int64, device=cuda_device))
    with pytest.raises(ValueError):
        m.infer(X, scores=torch.empty(10, 3, device=cuda_device))
    with pytest.raises(ValueError):
        m.infer_host(torch.randn(10, 19).pin_memory(), torch.empty(10, dtype=torch.int32).pin_memory())
    with pytest.raises(TypeError):
        m.infer_host(X.cpu().pin_memory(), torch.empty(10, dtype=torch.int64).pin_memory())
    with pytest.raises(ValueError):
        m.infer_host(X.cpu().pin_memory(), torch.empty(10, dtype=torch.int32, device=cuda_device))
    y, _ = m.infer(X)
    torch.cuda.synchronize()
    assert y.shape == (10,)
    m.close()
