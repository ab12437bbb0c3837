"""Helpers for the GPU parity tests (test infrastructure)."""
import numpy as np
import torch

import oracle
from oracle.policy import check_fp32, check_lowp

LOWP = ("tf32", "bf16")


def to_dev(*arrays):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrays]


def run_model(model, X, path="auto", scores=True):
    (Xd,) = to_dev(X)
    y, S = model.infer(Xd, path=path, return_scores=scores)
    torch.cuda.synchronize()
    return y.cpu().numpy(), (S.cpu().numpy() if S is not None else None)


def check_result(prec, kernel, X, B, C, y, S, north_star=True):
    """Judge one GPU result against the oracle by the arithmetic that produced it
    (DESIGN.md §3): the fp32 policy for fp32 semantics and for the fp32 kernels a
    low-precision model may run on (small / FFMA: sign-exact, a stronger claim); for the
    tf32 / bf16 tensor-core kernel the low-precision policy against the exact problem
    (rigorous allowance; north_star's 1e-2 on BJ configs) AND the fp32 policy against
    the problem on rounded operands."""
    if prec in LOWP and kernel == "tc":
        exact, rounded = oracle.infer_lowp(X, B, C, prec, nthreads=0)
        return check_lowp(exact, y, S, rtol=1e-2 if north_star else None, rounded=rounded)
    assert kernel in ("small", "small_tc", "ffma", "tc", "none"), kernel
    orc = oracle.infer(X, B, C, allow=True, nthreads=0)
    return check_fp32(orc, y, S)


def parity(X, B, C, path="auto", prec="fp32", model=None, north_star=True):
    """Run X through a model of B, C (or `model`) and check it (check_result)."""
    import paper_2506_09282_b200 as hdc
    own = model is None
    if own:
        Bd, Cd = to_dev(B, C)
        model = hdc.Model(Bd, Cd, prec=prec)
    y, S = run_model(model, X, path=path)
    kernel = model.last_kernel()
    rep = check_result(model.prec, kernel, X, B, C, y, S, north_star=north_star)
    rep["kernel"] = kernel
    if own:
        model.close()
    return rep, y, S


def parity_fp32(X, B, C, path="auto", prec="fp32", model=None):
    """fp32-semantics parity; returns (report, labels, scores, oracle result)."""
    import paper_2506_09282_b200 as hdc
    assert prec in ("fp32", "fp32_tc")
    orc = oracle.infer(X, B, C, allow=True, nthreads=0)
    own = model is None
    if own:
        Bd, Cd = to_dev(B, C)
        model = hdc.Model(Bd, Cd, prec=prec)
    y, S = run_model(model, X, path=path)
    rep = check_fp32(orc, y, S)
    if own:
        model.close()
    return rep, y, S, orc
