"""Shared helpers for the GPU-vs-oracle parity tests (tests only)."""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle
import paper_2602_10056_b200 as wc
from paper_2602_10056_b200.inputs import make_qkv

TOL = {"f32": 1e-4, "bf16": 2e-2}  # north star: max |O_gpu - O_orc| / ||V||_max


def run_gpu(Q, K, V, r, seed=0, beta=None, clip=True, block=1, bins=1, **kw):
    dev = torch.device("cuda:0")
    Qd, Kd, Vd = Q.to(dev), K.to(dev), V.to(dev)
    units = K.shape[0] * K.shape[1]
    R = wc._binding.coreset_rows(K.shape[2], r, bins)[1]
    S = torch.empty(units, R, dtype=torch.int32, device=dev)
    reff = torch.empty(units, dtype=torch.int32, device=dev)
    O = wc.forward(Qd, Kd, Vd, r, seed=seed, beta=beta, clip=clip, S=S, r_eff=reff, block=block, bins=bins, **kw)
    torch.cuda.synchronize()
    return O.float().cpu().numpy().astype(np.float64), S.cpu().numpy(), reff.cpu().numpy()


def run_oracle(Q, K, V, r, seed=0, beta=None, clip=True, block=1, bins=1, **kw):
    return oracle.forward(Q.double().numpy(), K.double().numpy(), V.double().numpy(), r, seed=seed,
                          beta=beta, clip=clip, block=block, bins=bins, **kw)


def compare(Q, K, V, r, dtype, seed=0, beta=None, clip=True, allow_pivot_mismatch=0, block=1, bins=1, **kw):
    """kw: unit_offset / tau_one / recenter, passed to both sides."""
    Og, Sg, Rg = run_gpu(Q, K, V, r, seed, beta, clip, block, bins, **kw)
    res = run_oracle(Q, K, V, r, seed, beta, clip, block, bins, **kw)
    mism = int((Sg != res["S"]).any(axis=1).sum() + (Rg != res["r_eff"]).sum())
    assert mism <= allow_pivot_mismatch, f"{mism} units with pivot mismatch"
    vmax = float(np.abs(V.double().numpy()).max())
    err = float(np.abs(Og - res["O"]).max()) / vmax
    assert err <= TOL[dtype], f"max rel err {err:.3e} > {TOL[dtype]}"
    return dict(err=err, S=Sg, r_eff=Rg, O=Og, orc=res)


def qkv(batch, hq, hkv, m, n, d, dtype, family="G", seed=0, distinct=None):
    return make_qkv(batch, hq, hkv, m, n, d, dtype, family, seed, distinct)
