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
