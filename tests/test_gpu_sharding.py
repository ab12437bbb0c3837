"""Sharding layer with the real CUDA model and NCCL (world_size 1 on the one
GPU this environment provides): the plumbing runs end to end and matches the
unsharded call."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from hdc_inputs import CONFIGS, make_B, make_C, make_X
from tests.gpu_util import to_dev

pytestmark = pytest.mark.gpu

@pytest.fixture(autouse=True)
def _fp32_on_ffma(monkeypatch):
    # fp32 models in this module exercise the fp32 FFMA kernels (HDC_PREC_FP32 otherwise
    # runs on the int8 tensor-core kernels when eligible, tested elsewhere)
    monkeypatch.setenv("HDC_FP32_FFMA", "1")



@pytest.fixture(scope="module")
def nccl_group(cuda_device):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda_device)
    yield
    dist.destroy_process_group()


def test_nshard_and_dshard_world1(nccl_group):
    import paper_2506_09282_b200 as hdc
    from paper_2506_09282_b200.sharding import shard_d_infer, shard_n_infer
    cfg = CONFIGS["cfg1"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    Xd, Bd, Cd = to_dev(X, B, C)
    m = hdc.Model(Bd, Cd, prec="fp32_tc")
    y0, S0 = m.infer(Xd, return_scores=True)
    y1, S1 = shard_n_infer(m, Xd, cfg.N, return_scores=True)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1) and torch.equal(S0, S1)
    y2, S2 = shard_d_infer(m, Xd[:16], hdc.argmax, return_scores=True)
    y3, S3 = m.infer(Xd[:16], path="small", return_scores=True)
    torch.cuda.synchronize()
    assert torch.equal(y2, y3) and torch.equal(S2, S3)
    m.close()


def test_dshard_in_kernel_exchange_world1(nccl_group):
    # the in-kernel D-shard reduction over torch symmetric memory, one rank: the exchange
    # runs (store, signal, wait, sum of one slot) and equals the plain small-batch call
    import paper_2506_09282_b200 as hdc
    from paper_2506_09282_b200.sharding import DShardExchange
    cfg = CONFIGS["cfg3_n32"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    Xd, Bd, Cd = to_dev(X, B, C)
    m = hdc.Model(Bd, Cd, prec="fp32")
    xc = DShardExchange(32, cfg.K)
    for n in (1, 7, 32, 32, 3):                      # several epochs, both parities
        y, S = xc.infer(m, Xd[:n], return_scores=True)
        y0, S0 = m.infer(Xd[:n], path="small", return_scores=True)
        torch.cuda.synchronize()
        assert torch.equal(y, y0) and torch.equal(S, S0)
    m.close()


def _slot(buf, world, stride, parity, sender):
    sigpad = (world + 3) // 4 * 4
    off = sigpad + (parity * world + sender) * stride
    return buf[off:off + stride]


@pytest.mark.parametrize("Ns", [(1, 1, 1), (13, 13, 13), (32, 32, 32), (32, 5, 17, 1, 32)])
def test_dshard_exchange_two_ranks_simulated(cuda_device, Ns):
    # Rank 0 of a 2-rank exchange on one GPU, WITHOUT a second kernel: rank 1's partial and
    # its signal are placed in rank 0's buffer beforehand, so the kernel never waits on
    # another kernel.  Checks the rank-order sum, the stores into the peer buffer and the
    # signals, for both parities -- and with N changing from call to call on the same
    # buffers (slots are sized for 32 rows, so their offsets never depend on N).
    import paper_2506_09282_b200 as hdc
    cfg = CONFIGS["cfg3_n32"]
    X, B, C = make_X(cfg, 0, 32), make_B(cfg), make_C(cfg)
    Xd, Bd, Cd = to_dev(X, B, C)
    cut = 4996                                        # multiple of 4 (d_shard_slices alignment)
    ma = hdc.Model(Bd[:, :cut].contiguous(), Cd[:, :cut].contiguous(), prec="fp32")
    mb = hdc.Model(Bd[:, cut:].contiguous(), Cd[:, cut:].contiguous(), prec="fp32")
    W, K = 2, cfg.K
    nwords = hdc.dshard_exchange_bytes(32, K, W) // 4
    assert all(hdc.dshard_exchange_bytes(n, K, W) // 4 == nwords for n in (1, 7, 32))
    stride = (32 * K + 3) // 4 * 4                    # slot floats: N-independent
    bufs = [torch.zeros(nwords, dtype=torch.float32, device="cuda") for _ in range(W)]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    for epoch, N in enumerate(Ns, start=1):
        par = epoch & 1
        Sa = ma.partial_scores(Xd[:N])
        Sb = mb.partial_scores(Xd[:N])
        _slot(bufs[0], W, stride, par, 1)[:N * K] = Sb.reshape(-1)            # rank 1's partial
        bufs[0][:W].view(torch.int32)[1] = epoch                              # ... and its signal
        y, S = ma.infer_dshard(Xd[:N], ptrs, 0, W, epoch, return_scores=True)
        torch.cuda.synchronize()
        expect = Sa + Sb                                                      # rank order
        assert torch.equal(S, expect)
        assert torch.equal(y, hdc.argmax(expect))
        assert torch.equal(_slot(bufs[1], W, stride, par, 0)[:N * K], Sa.reshape(-1))   # sent to rank 1
        assert int(bufs[1][:W].view(torch.int32)[0]) == epoch                 # rank 1 signalled
        assert int(bufs[0][:W].view(torch.int32)[0]) == epoch
    # argument checks
    with pytest.raises(hdc.HDCError):
        ma.infer_dshard(Xd, ptrs, 2, W, 4)
    ma.close()
    mb.close()
