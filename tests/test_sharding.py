"""Sharding layer (paper_2506_09282_b200.sharding) on a world_size-2 gloo group
on CPU.  The per-rank compute is a test double that evaluates the CPU oracle
(the kernels need a GPU); what is under test is the partition arithmetic, the
padding of uneven shards and the gather / all-reduce plumbing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2506_09282_b200.sharding import NShardGather, d_shard_slices, shard_bounds, shard_d_infer, shard_n_infer


class OracleRankModel:
    """Test double with the Model interface, backed by the oracle (float64)."""

    def __init__(self, B, C):
        self.B, self.C = B, C

    def infer(self, X, return_scores=False):
        out = oracle.infer(X.numpy(), self.B, self.C)
        S = torch.from_numpy(out["S"])
        return torch.from_numpy(out["y"]), (S if return_scores else None)

    def partial_scores(self, X):
        return torch.from_numpy(oracle.infer(X.numpy(), self.B, self.C)["S"])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(N=37, F=23, D=150, K=5, seed=3):
    rng = np.random.default_rng(seed)
    X = rng.uniform(-1, 1, (N, F)).astype(np.float32)
    B = rng.standard_normal((F, D)).astype(np.float32)
    C = rng.standard_normal((K, D)).astype(np.float32)
    return X, B, C


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, B, C = _inputs()
        N, D = X.shape[0], B.shape[1]
        # N-shard
        lo, hi = shard_bounds(N, world, rank)
        y, S = shard_n_infer(OracleRankModel(B, C), torch.from_numpy(X[lo:hi]), N, return_scores=True)
        # D-shard
        dlo, dhi = d_shard_slices(D, world)[rank]
        m = OracleRankModel(np.ascontiguousarray(B[:, dlo:dhi]), np.ascontiguousarray(C[:, dlo:dhi]))
        yd, Sd = shard_d_infer(m, torch.from_numpy(X), lambda s: torch.argmax(s, dim=1).to(torch.int32),
                               return_scores=True)
        # the benchmark's gather: shard labels into the padded buffer, one all_gather
        g = NShardGather(N)
        yl, _ = OracleRankModel(B, C).infer(torch.from_numpy(X[lo:hi]))
        g.labels.copy_(yl)
        g.gather()
        q.put((rank, y.numpy(), S.numpy(), yd.numpy(), Sd.numpy(), g.result().numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_partition():
    for total in (0, 1, 7, 100, 10000):
        for world in (1, 2, 3, 8):
            for align in (1, 4, 80):
                b = [shard_bounds(total, world, r, align) for r in range(world)]
                assert b[0][0] == 0 and b[-1][1] == total
                for (l0, h0), (l1, h1) in zip(b[:-1], b[1:]):
                    assert h0 == l1 and l0 <= h0
                for lo, hi in b[:-1]:
                    assert lo % align == 0 and hi % align == 0
    # 10000 columns over 8 ranks in multiples of 4: 1248/1252-wide slices
    widths = [hi - lo for lo, hi in d_shard_slices(10000, 8)]
    assert sum(widths) == 10000 and all(w % 4 == 0 for w in widths)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_world2_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X, B, C = _inputs()
    full = oracle.infer(X, B, C)
    for rank, y, S, yd, Sd, yg in res:
        assert np.array_equal(yg, full["y"])          # NShardGather: every row, in order
        # N-shard: rows are independent -> bit-identical to one process
        assert np.array_equal(y, full["y"]) and np.array_equal(S, full["S"])
        # D-shard: sum of partial scores equals the full scores up to float64 rounding
        assert np.all(np.abs(Sd - full["S"]) <= 1e-12 * full["c1"][None, :])
        ok = (yd == full["y"]) | (full["margin"] < 1e-9)
        assert ok.all()
    # all ranks hold the same result
    assert all(np.array_equal(r[1], res[0][1]) and np.array_equal(r[3], res[0][3]) for r in res)
