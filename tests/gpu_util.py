"""Helpers for the GPU parity tests (test infrastructure)."""
import numpy as np
import torch

import oracle
from oracle.policy import check_fp32, check_lowp


def to_dev(*arrays):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrays]


def run_model(model, X, path="auto", scores=True):
    (Xd,) = to_dev(X)
    y, S = model.infer(Xd, path=path, return_scores=scores)
    torch.cuda.synchronize()
    return y.cpu().numpy(), (S.cpu().numpy() if S is not None else None)


def parity_fp32(X, B, C, path="auto", prec="fp32", model=None):
    import paper_2506_09282_b200 as hdc
    orc = oracle.infer(X, B, C, allow=True, nthreads=0)
    own = model is None
    if own:
        Bd, Cd = to_dev(B, C)
        model = hdc.Model(Bd, Cd, prec=prec)
    y, S = run_model(model, X, path=path)
    rep = check_fp32(orc, y, S) if prec in ("fp32", "fp32_tc") else check_lowp(orc, y, S)
    if own:
        model.close()
    return rep, y, S, orc
