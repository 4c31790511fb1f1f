"""Pins for the blocked (accelerated) RPCholesky oracle, wco_select_blocked (reading Z22).

The paper names accelerated RPCholesky as the oversampling route out of the
sequential pivot loop; what it must reproduce is the LAW of sequential
RPCholesky (Eq. 4: each pivot is drawn with probability
proportional to the current residual diagonal).  These tests pin it against
things other than itself:
  * b = 1 is the sequential sampler, bit for bit (same Philox counters);
  * on a tiny kernel matrix the empirical law of ordered pivot triples matches
    the closed-form RPC law computed by brute force (Schur complements), and the
    test has the power to reject the naive "accept every candidate" sampler;
  * L L^T = h~(K_S, K_S), non-negative residual, exhaustion at distinct keys,
    r = n reproduces exact attention (Prop.).
"""
import itertools
import math

import numpy as np
import pytest
from scipy import stats

from paper_2602_10056_b200.inputs import make_qkv


def _unit(family="G", n=300, d=16, seed=0, distinct=None):
    _, K, _ = make_qkv(1, 1, 1, 4, n, d, "f32", family, seed, distinct)
    return K[0, 0].double().numpy()


@pytest.mark.parametrize("family,seed", [("G", 0), ("C", 1), ("L", 2)])
def test_block_one_is_sequential(orc, family, seed):
    K = _unit(family, seed=seed)
    kbar, st = orc.prologue(K, K)
    a = orc.select(K, kbar, st["g"], st["mstar"], 40, seed=seed, unit=3)
    b = orc.select_blocked(K, kbar, st["g"], st["mstar"], 40, 1, seed=seed, unit=3)
    assert np.array_equal(a["S"], b["S"]) and a["r_eff"] == b["r_eff"]
    assert np.array_equal(a["L"], b["L"]) and np.array_equal(a["F"], b["F"]) and np.array_equal(a["p"], b["p"])
    assert b["nblocks"] == b["ncand"] == a["r_eff"]


def test_accept_uniform_stream_is_distinct(orc):
    u = [orc.pivot_uniform(7, c, 2) for c in range(64)]
    v = [orc.accept_uniform(7, c, 2) for c in range(64)]
    assert len(set(u) & set(v)) == 0
    assert all(0.0 <= x < 1.0 for x in v)


def _rpc_law(H, r):
    """Closed-form law of ordered RPCholesky pivot sequences (Eq. 4): product over rounds of
    residual_diag[s_k] / trace(residual), residual = H - H[:,S] H[S,S]^-1 H[S,:]."""
    n = H.shape[0]
    law = {}
    for seq in itertools.permutations(range(n), r):
        pr = 1.0
        for k in range(r):
            S = list(seq[:k])
            if S:
                R = H - H[:, S] @ np.linalg.solve(H[np.ix_(S, S)], H[S, :])
            else:
                R = H
            dg = np.clip(np.diag(R), 0, None)
            pr *= dg[seq[k]] / dg.sum()
        law[seq] = pr
    return law


def _naive_law(H, r, b):
    """Law of the WRONG sampler that accepts every distinct candidate of a block (no rejection)
    for the first block of size b >= r: pivots are i.i.d. draws from diag(H) conditioned on
    distinctness.  Used only to show the test has power."""
    n = H.shape[0]
    dg = np.diag(H) / np.trace(H)
    law = {}
    for seq in itertools.permutations(range(n), r):
        pr, left = 1.0, 1.0
        for k in range(r):
            pr *= dg[seq[k]] / left
            left -= dg[seq[k]]
        law[seq] = pr
    return law


def _chi2(counts, law, N):
    keys = list(law)
    exp = np.array([law[k] * N for k in keys])
    obs = np.array([counts.get(k, 0) for k in keys], dtype=float)
    big = exp >= 5
    o = np.append(obs[big], obs[~big].sum())
    e = np.append(exp[big], exp[~big].sum())
    if e[-1] == 0:
        o, e = o[:-1], e[:-1]
    stat = float(((o - e) ** 2 / e).sum())
    return stat, len(o) - 1, big, exp


@pytest.mark.parametrize("sampler,b", [("blocked", 2), ("blocked", 4), ("blocked", 8), ("sequential", 1)])
def test_pivot_law_matches_brute_force_rpc(orc, sampler, b):
    rng = np.random.Generator(np.random.PCG64(42))
    n, d, r, N = 6, 3, 3, 20000
    K = rng.standard_normal((n, d))
    K[1] = K[0] + 0.05 * rng.standard_normal(d)  # a near-duplicate pair: strongly non-uniform conditionals
    g, mstar, kbar = 0.8, 0.0, np.zeros(d)
    H = np.exp(g * (K @ K.T) - mstar)
    law = _rpc_law(H, r)
    counts = {}
    for seed in range(N):
        if sampler == "sequential":
            S = orc.select(K, kbar, g, mstar, r, seed=seed)["S"]
        else:
            S = orc.select_blocked(K, kbar, g, mstar, r, b, seed=seed)["S"]
        key = tuple(int(x) for x in S)
        counts[key] = counts.get(key, 0) + 1
    assert set(counts) <= set(law)
    stat, dof, big, exp = _chi2(counts, law, N)
    pval = stats.chi2.sf(stat, dof)
    assert pval > 1e-4, (stat, dof, pval)
    # power: the naive no-rejection sampler would be rejected by a wide margin
    naive = _naive_law(H, r, b)
    nc = sum(N * (naive[k] - law[k]) ** 2 / law[k] for k in law if law[k] * N >= 5)
    assert stats.chi2.sf(nc, dof) < 1e-12


def test_blocked_factor_and_residual_invariants(orc):
    K = _unit("C", n=400, d=16, seed=5)
    kbar, st = orc.prologue(K, K)
    res = orc.select_blocked(K, kbar, st["g"], st["mstar"], 48, 16, seed=5, unit=1)
    S, re = res["S"], res["r_eff"]
    assert re == 48 and len(set(S.tolist())) == 48
    L = res["L"][:re, :re]
    Hs = orc.kernel_block(K[S], K[S], kbar, st["g"], st["mstar"])
    assert np.abs(L @ L.T - Hs).max() <= 1e-10 * np.abs(Hs).max()
    assert np.all(np.triu(L, 1) == 0) and np.all(np.diag(L) > 0)
    assert np.all(res["p"] >= 0) and np.all(res["p"][S] == 0)
    # residual diagonal = diag(H - F^T F) (Nystrom residual on every key)
    Hd = np.exp(st["g"] * ((K - kbar) ** 2).sum(1) - st["mstar"])
    assert np.abs(res["p"] - np.clip(Hd - (res["F"] ** 2).sum(0), 0, None)).max() <= 1e-10
    assert res["nblocks"] * 16 == res["ncand"] and res["ncand"] >= re


def test_blocked_exhaustion_distinct_keys(orc):
    K = _unit("D", n=500, d=16, seed=4, distinct=7)
    kbar, st = orc.prologue(K, K)
    res = orc.select_blocked(K, kbar, st["g"], st["mstar"], 20, 8, seed=4)
    assert res["r_eff"] == 7
    assert len({tuple(K[s]) for s in res["S"][:7]}) == 7 and np.all(res["S"][7:] == -1)


def test_blocked_full_rank_is_exact_attention(orc):
    rng = np.random.Generator(np.random.PCG64(9))
    n, d = 40, 8
    Q, K, V = (rng.standard_normal((n, d)) for _ in range(3))
    res = orc.forward(Q[None, None], K[None, None], V[None, None], n, seed=3, block=8, clip=False)
    ex = orc.exact_attention(Q, K, V)
    assert res["r_eff"][0] == n
    assert np.abs(res["O"][0, 0] - ex).max() <= 1e-8 * np.abs(V).max()
