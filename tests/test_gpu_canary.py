"""Out-of-bounds write detection without compute-sanitizer (closed on this GPU pool, see
profiles/round2/sanitizer/): every output the C ABI writes lives inside a larger buffer whose
margins hold a sentinel pattern; after the call the margins must be intact, the inputs must
be bit-identical, and the outputs must still pass the oracle.  Ragged shapes on every path,
precision and cluster shape."""
import numpy as np
import pytest
import torch

from tests.gpu_util import check_result

pytestmark = pytest.mark.gpu
PAD = 4096
SENT_F = -12345.678
SENT_I = -987654


@pytest.fixture(scope="module")
def hdc(cuda_device):
    import paper_2506_09282_b200 as pkg
    pkg.lib()
    return pkg


def _padded(n, dtype, sentinel):
    buf = torch.full((n + 2 * PAD,), sentinel, dtype=dtype, device="cuda")
    return buf, buf[PAD:PAD + n]


def _margins_ok(buf, n, sentinel):
    b = buf.cpu()
    return bool(torch.all(b[:PAD] == sentinel)) and bool(torch.all(b[PAD + n:] == sentinel))


CASES = [  # (prec, path, N, F, D, K, cluster)
    ("fp32_tc", "fused", 129, 61, 333, 7, None), ("fp32_tc", "fused", 5, 700, 1001, 26, None),
    ("fp32_tc", "fused", 300, 130, 167, 3, "1x4v"), ("bf16", "fused", 257, 33, 481, 32, None),
    ("bf16", "fused", 200, 64, 250, 5, "2x1p"), ("tf32", "fused", 140, 17, 97, 64, None),
    ("fp32", "fused", 131, 75, 300, 10, None), ("fp32", "small", 31, 90, 515, 6, None),
    ("fp32_tc", "small", 17, 784, 1234, 10, None), ("fp32_tc", "small", 3, 5, 9, 2, None),
    ("bf16", "small", 8, 100, 700, 4, None), ("fp32_tc", "auto", 1, 1, 1, 1, None),
    ("fp32", "fused", 131, 75, 300, 10, "ffma"), ("fp32", "small", 31, 90, 515, 6, "ffma"),
    ("fp32", "small", 9, 3000, 300, 6, "ffma"),
]


@pytest.mark.parametrize("prec,path,N,F,D,K,cluster", CASES)
def test_outputs_stay_in_bounds(hdc, monkeypatch, prec, path, N, F, D, K, cluster):
    if cluster == "ffma":
        monkeypatch.setenv("HDC_FP32_FFMA", "1")       # the fp32 FFMA / streaming kernels
    elif cluster:
        monkeypatch.setenv("HDC_TC_CLUSTER", cluster)
    monkeypatch.setenv("HDC_SMALL_TC", "1")
    rng = np.random.default_rng(N * 31 + F * 7 + D + K)
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    xbuf, Xd = _padded(N * F, torch.float32, SENT_F)
    Xd.copy_(torch.from_numpy(X).reshape(-1))
    Bd, Cd = torch.from_numpy(B).cuda(), torch.from_numpy(C).cuda()
    m = hdc.Model(Bd, Cd, prec=prec)
    lbuf, labels = _padded(N, torch.int32, SENT_I)
    sbuf, scores = _padded(N * K, torch.float32, SENT_F)
    for _ in range(2):                                 # second call: workspaces reused
        m.infer(Xd.view(N, F), labels=labels, scores=scores.view(N, K), path=path)
    torch.cuda.synchronize()
    kernel = m.last_kernel()
    assert _margins_ok(lbuf, N, SENT_I) and _margins_ok(sbuf, N * K, SENT_F), (prec, path, kernel)
    assert _margins_ok(xbuf, N * F, SENT_F) and np.array_equal(Xd.cpu().numpy(), X.reshape(-1))
    check_result(prec, kernel, X, B, C, labels.cpu().numpy(), scores.view(N, K).cpu().numpy(), north_star=False)
    # labels only (scores NULL): the kernels' own scratch, nothing outside
    lbuf2, labels2 = _padded(N, torch.int32, SENT_I)
    m.infer(Xd.view(N, F), labels=labels2, path=path)
    torch.cuda.synchronize()
    assert _margins_ok(lbuf2, N, SENT_I) and torch.equal(labels2, labels)
    m.close()


def test_encode_and_host_path_stay_in_bounds(hdc):
    rng = np.random.default_rng(3)
    N, F, D, K = 77, 50, 333, 5
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    m = hdc.Model(torch.from_numpy(B).cuda(), torch.from_numpy(C).cuda(), prec="fp32_tc")
    ldw = (D + 31) // 32
    hbuf = torch.full((N * ldw + 2 * PAD,), SENT_I, dtype=torch.int32, device="cuda")
    H = hbuf[PAD:PAD + N * ldw].view(N, ldw)
    m.encode(torch.from_numpy(X).cuda(), H=H)
    torch.cuda.synchronize()
    assert _margins_ok(hbuf, N * ldw, SENT_I)
    lh = torch.full((N + 2 * PAD,), SENT_I, dtype=torch.int32).pin_memory()
    sh = torch.full((N * K + 2 * PAD,), SENT_F, dtype=torch.float32).pin_memory()
    m.infer_host(torch.from_numpy(X).pin_memory(), lh[PAD:PAD + N], sh[PAD:PAD + N * K])
    torch.cuda.synchronize()
    assert bool(torch.all(lh[:PAD] == SENT_I)) and bool(torch.all(lh[PAD + N:] == SENT_I))
    assert bool(torch.all(sh[:PAD] == SENT_F)) and bool(torch.all(sh[PAD + N * K:] == SENT_F))
    m.close()
