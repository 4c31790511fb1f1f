"""Pins for the oracle's weights, weighted attend and exact attention.

Against: the hand-evaluated Eq. 1 example (tests/golden/paper_constants.txt),
closed forms (n = 1, beta = 0, r = 1), exactness of full-rank / distinct-key
Nystrom, numpy pseudo-inverse Nystrom weights, and Lemma 2.1
 as a zero-violation theorem check.
"""
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _g(shape, seed, scale=1.0):
    return scale * np.random.Generator(np.random.PCG64(seed)).standard_normal(shape)


def _consts():
    out = {}
    with open(os.path.join(GOLDEN, "paper_constants.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            name, val, tol = line.split()[:3]
            out[name] = ([float(x) for x in val.split(",")], float(tol))
    return out


def test_exact_attention_hand_example(orc):
    c = _consts()
    Q = np.array([[1.0], [-1.0]])
    V = np.eye(2)
    O = np.zeros((2, 2))
    # d = 1 but V has 2 columns: evaluate each column with a 1-column V
    for col in range(2):
        O[:, col] = orc.exact_attention(Q, Q, V[:, [col]], beta=1.0)[:, 0]
    for i, key in enumerate(["exact_hand_row0", "exact_hand_row1"]):
        want, tol = c[key]
        assert np.abs(O[i] - np.array(want)).max() <= tol


def test_exact_attention_closed_forms(orc):
    Q, K, V = _g((20, 6), 1), _g((30, 6), 2), _g((30, 6), 3)
    # beta = 0: uniform weights -> column mean
    assert np.abs(orc.exact_attention(Q, K, V, beta=0.0) - V.mean(0)).max() < 1e-14
    # n = 1: every row equals the single value row
    assert np.abs(orc.exact_attention(Q, K[:1], V[:1]) - V[0]).max() < 1e-15
    # convex combination: inside the columnwise value range
    O = orc.exact_attention(Q, K, V)
    assert np.all(O >= V.min(0) - 1e-15) and np.all(O <= V.max(0) + 1e-15)
    # recentring invariance
    O2 = orc.exact_attention(Q, K + _g((1, 6), 4), V)
    assert np.abs(O - O2).max() < 1e-12


def _wildcat(orc, Q, K, V, r, seed=0, beta=None, clip=True):
    res = orc.forward(Q[None, None], K[None, None], V[None, None], r, seed=seed, beta=beta, clip=clip)
    return res["O"][0, 0], res


def test_weights_match_pinv_definition(orc):
    # X = W [V, 1] with W = h(K_S,K_S)^+ h(K_S,K), numpy pinv (SVD)
    n, d, r = 90, 8, 14
    K, V = _g((n, d), 5), _g((n, d), 6)
    kbar, st = orc.prologue(K, _g((20, d), 7))
    f = orc.select(K, kbar, st["g"], st["mstar"], r, seed=1)
    S = list(f["S"])
    X = orc.weights(K, V, f["S"], f["r_eff"], kbar, st["g"], st["mstar"])
    H = orc.kernel_block(K, K, kbar, st["g"], st["mstar"])
    W = np.linalg.pinv(H[np.ix_(S, S)], rcond=1e-15) @ H[S, :]
    Xref = W @ np.hstack([V, np.ones((n, 1))])
    cond = np.linalg.cond(H[np.ix_(S, S)])
    assert np.abs(X - Xref).max() <= 1e-12 * cond * max(1.0, np.abs(Xref).max())
    # and against the literal Alg 1 weights W = M R
    a = orc.select_mr(K, kbar, st["g"], st["mstar"], r, seed=1)
    assert np.abs(X - a["W"] @ np.hstack([V, np.ones((n, 1))])).max() <= 1e-12 * cond * np.abs(Xref).max()


@pytest.mark.parametrize("seed", range(5))
def test_full_rank_is_exact(orc, seed):
    # r = n: the Nystrom approximation is exact (SPEC.md acceptance 2)
    n, d = 24, 6
    Q, K, V = _g((n, d), 10 + seed), _g((n, d), 20 + seed), _g((n, d), 30 + seed)
    O = orc.exact_attention(Q, K, V)
    Oh, res = _wildcat(orc, Q, K, V, r=n, seed=seed)
    assert np.abs(Oh - O).max() <= 1e-6 * np.abs(V).max()


@pytest.mark.parametrize("seed", range(4))
def test_distinct_keys_exact(orc, seed):
    # keys from m distinct vectors, r >= m: exact attention (north star)
    mdist, n, d = 5, 80, 8
    base = _g((mdist, d), 40 + seed)
    idx = np.random.Generator(np.random.PCG64(seed)).integers(0, mdist, n)
    K = base[idx]
    Q, V = _g((50, d), 50 + seed), _g((n, d), 60 + seed)
    Oh, res = _wildcat(orc, Q, K, V, r=12, seed=seed)
    assert res["r_eff"][0] == mdist
    assert np.abs(Oh - orc.exact_attention(Q, K, V)).max() <= 1e-10 * np.abs(V).max()


def test_rank_one_is_query_independent(orc):
    n, d = 60, 8
    Q, K, V = _g((40, d), 1), _g((n, d), 2), _g((n, d), 3)
    Oh, res = _wildcat(orc, Q, K, V, r=1, seed=4, clip=False)
    X = res["X"][0]
    assert np.abs(Oh - X[0, :d] / X[0, d]).max() < 1e-13


def test_beta_to_zero_gives_mean(orc):
    n, d = 70, 8
    Q, K, V = _g((30, d), 1), _g((n, d), 2), _g((n, d), 3)
    Oh, res = _wildcat(orc, Q, K, V, r=8, seed=0, beta=1e-14)
    assert res["r_eff"][0] == 1
    assert np.abs(Oh - V.mean(0)).max() < 1e-10


def test_single_key_returns_value(orc):
    Q, K, V = _g((5, 4), 1), _g((1, 4), 2), _g((1, 4), 3)
    Oh, res = _wildcat(orc, Q, K, V, r=1)
    assert np.abs(Oh - V[0]).max() < 1e-14


def test_clip_range_and_zero_denominator(orc):
    n, d, r = 100, 8, 10
    Q, K, V = _g((64, d), 1, 3.0), _g((n, d), 2, 3.0), _g((n, d), 3)
    Oh, _ = _wildcat(orc, Q, K, V, r=r, seed=2)
    assert np.all(Oh >= V.min(0)) and np.all(Oh <= V.max(0))
    # den <= 0 rows produce clip(0): a cache with w < 0 everywhere
    KS = K[:2]
    X = np.hstack([np.ones((2, d)), -np.ones((2, 1))])
    O = orc.attend(Q, KS, X, 2, 0.3, V.min(0), V.max(0), clip=True)
    assert np.abs(O - np.clip(0.0, V.min(0), V.max(0))).max() == 0.0


def test_lemma21_bound_zero_violations(orc):
    # Lemma 2.1: ||O - O^||_max <= ||V||_max min(3 ||A - A^||_{2->inf} / (sqrt(n) min A), 2)
    # for the plug-in estimator with A^ = h(Q, K_S) W (W from the literal Alg 1).
    violations = 0
    for t in range(30):
        rng = np.random.Generator(np.random.PCG64(t))
        n, m, d = int(rng.integers(8, 48)), int(rng.integers(4, 40)), int(rng.integers(2, 8))
        r = int(rng.integers(1, n + 1))
        Q, K, V = rng.standard_normal((m, d)), rng.standard_normal((n, d)), rng.standard_normal((n, d))
        beta = 1 / math.sqrt(d)
        Oh, res = _wildcat(orc, Q, K, V, r=r, seed=t)
        kbar, st = orc.prologue(K, Q)
        a = orc.select_mr(K, kbar, st["g"], st["mstar"], r, seed=t, unit=0)
        S = list(a["S"][: a["r_eff"]])
        A = np.exp(beta * Q @ K.T)
        Ahat = np.exp(beta * Q @ K[S].T) @ a["W"][: a["r_eff"]]
        O = orc.exact_attention(Q, K, V)
        lhs = np.abs(O - Oh).max()
        if lhs > orc.lemma21_rhs(A, Ahat, V) + 1e-9 * np.abs(V).max():
            violations += 1
    assert violations == 0


def test_error_decreases_with_rank(orc):
    # Mean max-norm error at r = 64 is below r = 8 (Theorem 2.3 direction; SPEC acceptance 7, loose)
    errs = {8: [], 64: []}
    for seed in range(4):
        n, d = 256, 8
        Q, K, V = _g((n, d), seed, 0.5), _g((n, d), 100 + seed, 0.5), _g((n, d), 200 + seed)
        O = orc.exact_attention(Q, K, V)
        for r in errs:
            Oh, _ = _wildcat(orc, Q, K, V, r=r, seed=seed)
            errs[r].append(np.abs(O - Oh).max())
    assert np.mean(errs[64]) <= 0.5 * np.mean(errs[8])


def test_gqa_forward_groups(orc):
    # two query heads share one kv head: R_Q over the group (Alg 4, reading Z11)
    d = 8
    Q = _g((1, 2, 30, d), 1)
    K, V = _g((1, 1, 50, d), 2), _g((1, 1, 50, d), 3)
    res = orc.forward(Q, K, V, 10, seed=5)
    rq = np.sqrt((Q[0].reshape(-1, d) ** 2).sum(1)).max()
    assert res["stats"][0, 4] == pytest.approx(rq, rel=1e-15)
    for h in range(2):
        KS = K[0, 0][res["S"][0]]
        O = orc.attend(Q[0, h], KS, res["X"][0], res["r_eff"][0], 1 / math.sqrt(d),
                       V[0, 0].min(0), V[0, 0].max(0))
        assert np.abs(O - res["O"][0, h]).max() == 0.0
