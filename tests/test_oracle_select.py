"""Pins for the oracle's RPNys selection (Alg 1; Eq. 4).

Checks against: brute-force enumeration of the pivot-sequence law from the plain
residual diag(H - H_{:,S} H_SS^{-1} H_{S,:}) (numpy solve), the first-pivot example
of SPEC.md:255, the literal M/R form of Alg 1 (Prop. PAPER.md:1757-1821), the
direct Nystrom residual, and exact structural properties.
"""
import itertools
import math

import numpy as np
import pytest
from scipy.stats import chisquare


def _gauss(n, d, seed, scale=1.0):
    return scale * np.random.Generator(np.random.PCG64(seed)).standard_normal((n, d))


def _seq_prob(H, seq):
    """Probability of drawing the ordered pivot sequence `seq` under Eq. 4, with the
    residual computed directly from its definition (h_res = h - h_nys)."""
    prob = 1.0
    S = []
    n = H.shape[0]
    for s in seq:
        if S:
            Hss = H[np.ix_(S, S)]
            Hks = H[:, S]
            res = np.diag(H) - np.einsum("ij,ij->i", Hks, np.linalg.solve(Hss, Hks.T).T)
        else:
            res = np.diag(H).copy()
        res[S] = 0.0
        res = np.maximum(res, 0.0)
        prob *= res[s] / res.sum()
        S.append(s)
    return prob


def test_pivot_sequence_law_bruteforce(orc):
    n, d, r = 5, 3, 3
    K = _gauss(n, d, 3, 0.8)
    kbar = np.zeros(d)
    g, mstar = 0.7, 0.0
    H = orc.kernel_block(K, K, kbar, g, mstar)
    seqs = list(itertools.permutations(range(n), r))
    probs = np.array([_seq_prob(H, s) for s in seqs])
    assert probs.sum() == pytest.approx(1.0, abs=1e-12)
    trials = 30000
    counts = {s: 0 for s in seqs}
    for seed in range(trials):
        res = orc.select(K, kbar, g, mstar, r, seed=seed, unit=5)
        counts[tuple(int(x) for x in res["S"])] += 1
    obs = np.array([counts[s] for s in seqs])
    exp = probs * trials
    # pool tiny cells for the chi-square approximation
    keep = exp >= 5
    obs_k = np.append(obs[keep], obs[~keep].sum())
    exp_k = np.append(exp[keep], exp[~keep].sum())
    stat, pval = chisquare(obs_k, exp_k)
    assert pval > 1e-3, (stat, pval)


def test_first_pivot_law_spec_example(orc):
    # two keys with kernel diagonal (1, 2): P(s = second) = 2/3.
    K = np.array([[0.0], [math.sqrt(math.log(2.0))]])
    hits = sum(int(orc.select(K, np.zeros(1), 1.0, 0.0, 1, seed=s)["S"][0] == 1) for s in range(20000))
    p = hits / 20000
    assert abs(p - 2 / 3) < 4 * math.sqrt((2 / 9) / 20000)


@pytest.mark.parametrize("seed", range(6))
def test_F_form_matches_literal_alg1(orc, seed):
    n, d, r = 64, 8, 16
    K = _gauss(n, d, 100 + seed)
    kbar, st = orc.prologue(K, _gauss(n, d, 200 + seed))
    f = orc.select(K, kbar, st["g"], st["mstar"], r, seed=seed, unit=2)
    a = orc.select_mr(K, kbar, st["g"], st["mstar"], r, seed=seed, unit=2)
    assert f["r_eff"] == a["r_eff"] == r
    assert np.array_equal(f["S"], a["S"])
    S = list(f["S"])
    H = orc.kernel_block(K, K, kbar, st["g"], st["mstar"])
    Hss = H[np.ix_(S, S)]
    # M = h(K_S,K_S)^{-1}  (Prop. "Recursive update of kernel inverse")
    Minv = np.linalg.inv(Hss)
    cond = np.linalg.cond(Hss)
    assert np.abs(a["M"] - Minv).max() <= 1e-12 * cond * np.abs(Minv).max()
    # W (Alg 1 output) = H_SS^{-1} H_SK  = L^{-T} F   (F = L^{-1} H_SK)
    W_direct = np.linalg.solve(Hss, H[S, :])
    assert np.abs(a["W"] - W_direct).max() <= 1e-10 * cond
    W_F = np.linalg.solve(f["L"].T, f["F"])
    assert np.abs(W_F - W_direct).max() <= 1e-10 * cond
    # final residual = diag(H - H_KS H_SS^{-1} H_SK)
    res = np.diag(H) - np.einsum("ij,ji->i", H[:, S], W_direct)
    assert np.abs(f["p"] - np.maximum(res, 0) * (np.arange(n)[:, None] != np.array(S)[None]).all(1)).max() <= 1e-12
    assert np.abs(a["p"] - f["p"]).max() <= 1e-13


def test_selection_invariants(orc):
    n, d, r = 300, 16, 40
    K = _gauss(n, d, 7) + 2.0
    kbar, st = orc.prologue(K, _gauss(50, d, 8))
    f = orc.select(K, kbar, st["g"], st["mstar"], r, seed=11)
    S = list(f["S"][: f["r_eff"]])
    assert len(set(S)) == len(S) == f["r_eff"] == r
    tr = f["trace"]
    assert np.all(np.diff(tr) <= 0)                # trace non-increasing
    assert np.all(f["p"] >= 0) and np.all(f["p"][S] == 0)
    L = f["L"]
    assert np.all(np.triu(L, 1) == 0)              # lower-triangular
    H = orc.kernel_block(K[S], K[S], kbar, st["g"], st["mstar"])
    assert np.abs(L @ L.T - H).max() <= 1e-12     # L is the Cholesky factor of H~_SS
    assert np.all(np.diag(L) > 0)
    # h~ in (0, 1]: diagonal of H~ bounded by 1 (Cauchy-Schwarz with R_K, reading Z10)
    assert tr[0] <= n * (1 + 1e-12)


def test_exhaustion_distinct_keys(orc):
    # keys drawn from m distinct vectors: the kernel matrix has rank m; after m pivots
    # the residual is (numerically) zero and selection stops with r_eff = m (reading Z3).
    mdist, n, d = 6, 120, 8
    base = _gauss(mdist, d, 1)
    idx = np.random.Generator(np.random.PCG64(2)).integers(0, mdist, n)
    idx[:mdist] = np.arange(mdist)
    K = base[idx]
    kbar, st = orc.prologue(K, _gauss(10, d, 3))
    for seed in range(5):
        f = orc.select(K, kbar, st["g"], st["mstar"], 20, seed=seed)
        assert f["r_eff"] == mdist
        assert sorted(idx[f["S"][:mdist]]) == list(range(mdist))
        assert np.all(f["S"][mdist:] == -1)


def test_single_key(orc):
    K = np.array([[0.3, -1.2, 0.5]])
    kbar, st = orc.prologue(K, K)
    # n = 1: the centred key is zero, R_K = 0, tau = 1 (fallback)
    assert st["tau"] == 1.0 and st["rk"] == 0.0
    a = orc.select_mr(K, kbar, st["g"], st["mstar"], 1, seed=0)
    assert list(a["S"]) == [0] and a["W"][0, 0] == pytest.approx(1.0, abs=1e-15)
    assert a["p"][0] == 0.0


def test_pivot_stream_depends_on_unit_and_seed(orc):
    n, d, r = 200, 8, 10
    K = _gauss(n, d, 4)
    kbar, st = orc.prologue(K, K)
    s00 = orc.select(K, kbar, st["g"], st["mstar"], r, seed=0, unit=0)["S"]
    assert np.array_equal(s00, orc.select(K, kbar, st["g"], st["mstar"], r, seed=0, unit=0)["S"])
    assert not np.array_equal(s00, orc.select(K, kbar, st["g"], st["mstar"], r, seed=0, unit=1)["S"])
    assert not np.array_equal(s00, orc.select(K, kbar, st["g"], st["mstar"], r, seed=1, unit=0)["S"])


def test_recentring_invariance_of_selection(orc):
    # compress_kv(K) and compress_kv(K + 1 c^T) see the same centred keys
    n, d, r = 150, 8, 12
    K = _gauss(n, d, 9)
    Q = _gauss(40, d, 10)
    k1, s1 = orc.prologue(K, Q)
    k2, s2 = orc.prologue(K + 0.75, Q)
    a = orc.select(K, k1, s1["g"], s1["mstar"], r, seed=3)
    b = orc.select(K + 0.75, k2, s2["g"], s2["mstar"], r, seed=3)
    assert s1["rk"] == pytest.approx(s2["rk"], rel=1e-12)
    assert np.array_equal(a["S"], b["S"])


def test_kbar_is_the_row_mean(orc):
    # Alg 2 "Recenter keys": kbar = (1/n) sum_l k_l, pinned directly (not only through
    # shift invariance): dyadic keys with n a power of two make the mean exact in fp64, so any other
    # centre (median, midrange, a dropped row, a 1/(n-1) scale) fails bit for bit.
    rng = np.random.default_rng(5)
    n, d = 256, 16
    K = rng.integers(-64, 64, size=(n, d)).astype(np.float64) / 8.0
    K[7] += 40.0  # an outlier row moves the mean but not the median
    kbar, st = orc.prologue(K, K[:10])
    assert np.array_equal(kbar, K.sum(0) / n)
    # R_K = max_l ||k_l - kbar||, R_Q = max_i ||q_i||, against numpy on the same data
    assert st["rk"] == pytest.approx(np.sqrt(((K - K.mean(0)) ** 2).sum(1)).max(), rel=1e-14)
    assert st["rq"] == pytest.approx(np.sqrt((K[:10] ** 2).sum(1)).max(), rel=1e-14)
    # Gaussian keys: within a few ulps of the compensated mean
    G = rng.standard_normal((1000, 8))
    kg, _ = orc.prologue(G, G[:5])
    exact = np.array([math.fsum(G[:, j]) / 1000 for j in range(8)])
    assert np.abs(kg - exact).max() <= 1e-15 * np.abs(G).max()
