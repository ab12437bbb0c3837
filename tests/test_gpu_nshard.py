"""N-shard invariance (SURVEY §8e exact test) on one GPU: the rows of a BASELINE batch split
into g = 2/4/8 contiguous shards (sharding.shard_bounds, ScalableHD-L row ownership P:410),
each shard inferred on its own as a rank would, the shard outputs concatenated as the label
all-gather does.  The fused tensor-core kernel sums every row's Stage II tiles exactly (int64
fixed point), so shard results equal the one-batch results BIT FOR BIT -- whatever the split,
the cluster shape or the tile schedule -- and the one-batch result is checked against the
oracle on every row elsewhere (test_gpu_tc.py)."""
import numpy as np
import pytest
import torch

from hdc_inputs import CONFIGS, make_B, make_C, make_X
from hdc_inputs.device import make_X_device
from paper_2506_09282_b200.sharding import shard_bounds
from tests.gpu_util import check_result, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hdc(cuda_device):
    import paper_2506_09282_b200 as pkg
    pkg.lib()
    return pkg


def _sharded(model, Xd, g, path="fused"):
    N = Xd.shape[0]
    ys, Ss = [], []
    for r in range(g):
        lo, hi = shard_bounds(N, g, r)
        y, S = model.infer(Xd[lo:hi], path=path, return_scores=True)
        ys.append(y)
        Ss.append(S)
    torch.cuda.synchronize()
    return torch.cat(ys).cpu().numpy(), torch.cat(Ss).cpu().numpy()


@pytest.mark.parametrize("prec", ["fp32_tc", "bf16", "tf32"])
def test_cfg2_shards_bitwise_equal_one_batch(hdc, prec):
    cfg = CONFIGS["cfg2"]
    B, C = make_B(cfg), make_C(cfg)
    Bd, Cd = to_dev(B, C)
    Xd = make_X_device(cfg, torch.device("cuda:0"))
    m = hdc.Model(Bd, Cd, prec=prec)
    y1, S1 = m.infer(Xd, return_scores=True)
    torch.cuda.synchronize()
    y1, S1 = y1.cpu().numpy(), S1.cpu().numpy()
    assert m.last_kernel() == "tc"
    for g in (2, 4, 8):
        yg, Sg = _sharded(m, Xd, g)
        assert np.array_equal(Sg, S1), (prec, g, np.abs(Sg - S1).max())
        assert np.array_equal(yg, y1)
    m.close()


@pytest.mark.parametrize("prec", ["fp32_tc", "bf16"])
def test_uneven_shards_and_oracle(hdc, prec):
    # shards that are not multiples of the 128-row tile (cfg1: 256 rows into 3 and 5), and the
    # smallest shards on the fused kernel (the split-N-tile path: one tile spread over many
    # CTAs); the concatenation is checked against the oracle on every row
    cfg = CONFIGS["cfg1"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    Xd, Bd, Cd = to_dev(X, B, C)
    m = hdc.Model(Bd, Cd, prec=prec)
    y1, S1 = m.infer(Xd, path="fused", return_scores=True)
    torch.cuda.synchronize()
    y1, S1 = y1.cpu().numpy(), S1.cpu().numpy()
    for g in (3, 5, 32, 64):
        yg, Sg = _sharded(m, Xd, g)
        assert np.array_equal(Sg, S1) and np.array_equal(yg, y1), (prec, g)
    rep = check_result(prec, "tc", X, B, C, yg, Sg)
    print(prec, rep)
    m.close()


@pytest.mark.parametrize("shape", ["1x1", "1x2", "2x1p", "1x4v"])
def test_cluster_shapes_bitwise_equal(hdc, monkeypatch, shape):
    # the same rows on every cluster shape / virtual group / CTA pair: identical scores
    cfg = CONFIGS["cfg1"]
    X, B, C = make_X(cfg), make_B(cfg), make_C(cfg)
    Xd, Bd, Cd = to_dev(X, B, C)
    out = {}
    for sh in ("2x1", shape):
        monkeypatch.setenv("HDC_TC_CLUSTER", sh)
        m = hdc.Model(Bd, Cd, prec="bf16")
        y, S = m.infer(Xd, path="fused", return_scores=True)
        torch.cuda.synchronize()
        out[sh] = (y.cpu().numpy(), S.cpu().numpy())
        m.close()
    assert np.array_equal(out[shape][1], out["2x1"][1]) and np.array_equal(out[shape][0], out["2x1"][0])
