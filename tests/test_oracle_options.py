"""Pins for the oracle's options: the PAR2 unit offset (Philox unit ids, reading Z2)
and the prologue switches WC_TAU_ONE / WC_NO_RECENTER (Alg 2).

Checks against: the batch run itself (a partition must reproduce it bit for bit), keys whose mean is
exactly zero (recentring by an exact zero is the identity), the plain kernel definition evaluated with
numpy on the selected pivots (L L^T = h(K_S, K_S), P:306 at tau = 1), closed forms of tau, g, mstar and
R_K, and exactness (r = n reproduces Eq. 1 attention, whatever kernel is used to select).
"""
import numpy as np
import pytest

from paper_2602_10056_b200.inputs import make_qkv


def _f64(*ts):
    return [t.double().numpy() for t in ts]


@pytest.mark.parametrize("block,bins", [(1, 1), (8, 1), (1, 4), (4, 2)])
def test_unit_offset_partition_is_bitwise_the_batch(orc, block, bins):
    """A GPU holding units [u0, u0 + U) with unit_offset = u0 selects the batch run's pivots (PAR2)."""
    Q, K, V = _f64(*make_qkv(2, 4, 2, 40, 96, 16, "f32", "G", 3))
    full = orc.forward(Q, K, V, 12, seed=5, block=block, bins=bins)
    # units are (batch, kv-head) = b * hkv + h: the second batch element is units 2, 3
    part = orc.forward(Q[1:], K[1:], V[1:], 12, seed=5, block=block, bins=bins, unit_offset=2)
    assert np.array_equal(full["S"][2:], part["S"])
    assert np.array_equal(full["r_eff"][2:], part["r_eff"])
    assert np.array_equal(full["O"][1:], part["O"])
    # and without the offset the streams differ (the offset is what reproduces the batch)
    wrong = orc.forward(Q[1:], K[1:], V[1:], 12, seed=5, block=block, bins=bins)
    assert not np.array_equal(full["S"][2:], wrong["S"])


def test_unit_offset_matches_select_unit_id(orc):
    """unit_offset = u0 draws the stream of unit id u0 of wco_select (pinned by the pivot-law tests)."""
    Q, K, V = _f64(*make_qkv(1, 1, 1, 30, 80, 8, "f32", "G", 4))
    res = orc.forward(Q, K, V, 10, seed=9, unit_offset=77)
    kbar, st = orc.prologue(K[0, 0], Q[0, 0])
    sel = orc.select(K[0, 0], kbar, st["g"], st["mstar"], 10, seed=9, unit=77)
    assert np.array_equal(res["S"][0], sel["S"])


def test_no_recenter_equals_default_when_mean_is_exactly_zero(orc):
    """Keys interleaved as (a_1, -a_1, a_2, -a_2, ...): every even prefix sum is exactly 0, so the
    default's kbar is exactly 0 and recentring is the identity -- bit-equal to WC_NO_RECENTER."""
    rng = np.random.Generator(np.random.PCG64(11))
    n, d, m = 64, 16, 24
    A = rng.standard_normal((n // 2, d))
    K = np.empty((n, d))
    K[0::2], K[1::2] = A, -A
    K = K[None, None]
    Q = rng.standard_normal((1, 1, m, d))
    V = rng.standard_normal((1, 1, n, d))
    kbar, _ = orc.prologue(K[0, 0], Q[0, 0])
    assert np.all(kbar == 0.0)
    a = orc.forward(Q, K, V, 10, seed=2)
    b = orc.forward(Q, K, V, 10, seed=2, recenter=False)
    assert np.array_equal(a["S"], b["S"]) and np.array_equal(a["O"], b["O"])


def test_no_recenter_stats_closed_form(orc):
    """kbar = 0 and R_K = max ||k_l|| on the uncentred keys (P:304 without P:300-301)."""
    Q, K, V = _f64(*make_qkv(1, 1, 1, 20, 50, 8, "f32", "L", 6))
    kbar, st = orc.prologue(K[0, 0], Q[0, 0], recenter=False)
    assert np.all(kbar == 0.0)
    assert st["rk"] == pytest.approx(np.linalg.norm(K[0, 0], axis=1).max(), rel=1e-14)
    kbar_c, st_c = orc.prologue(K[0, 0], Q[0, 0])
    assert st_c["rk"] == pytest.approx(np.linalg.norm(K[0, 0] - K[0, 0].mean(0), axis=1).max(), rel=1e-14)
    assert st["rk"] > st_c["rk"]  # the L family has a large per-channel offset


@pytest.mark.parametrize("recenter", [True, False])
def test_tau_one_kernel_is_the_untempered_softmax_kernel(orc, recenter):
    """WC_TAU_ONE: tau = 1, g = beta, mstar = beta R_K^2, and the selection's Cholesky factor
    satisfies L L^T = exp(beta <k_a - kbar, k_b - kbar> - mstar) on the pivots (numpy)."""
    Q, K, V = _f64(*make_qkv(1, 1, 1, 30, 70, 8, "f32", "G", 8))
    beta = 0.9
    kbar, st = orc.prologue(K[0, 0], Q[0, 0], beta=beta, tau_one=True, recenter=recenter)
    assert st["tau"] == 1.0 and st["g"] == beta
    assert st["mstar"] == pytest.approx(beta * st["rk"] ** 2, rel=1e-15)
    sel = orc.select(K[0, 0], kbar, st["g"], st["mstar"], 12, seed=3)
    re = sel["r_eff"]
    KS = K[0, 0][sel["S"][:re]] - kbar
    H = np.exp(beta * KS @ KS.T - st["mstar"])
    L = sel["L"][:re, :re]
    assert np.abs(L @ L.T - H).max() <= 1e-13 * np.abs(H).max()
    # the tempered default is a different kernel (tau from Eq. 7 is not 1 here)
    _, st_t = orc.prologue(K[0, 0], Q[0, 0], beta=beta, recenter=recenter)
    assert st_t["tau"] != 1.0


@pytest.mark.parametrize("tau_one,recenter", [(True, True), (False, False), (True, False)])
def test_options_full_rank_is_exact_attention(orc, tau_one, recenter):
    """r = n reproduces exact softmax attention (Eq. 1) with any selection kernel."""
    Q, K, V = _f64(*make_qkv(1, 2, 1, 16, 24, 8, "f32", "G", 12))
    res = orc.forward(Q, K, V, 24, seed=1, tau_one=tau_one, recenter=recenter, clip=False)
    for h in range(2):
        ex = orc.exact_attention(Q[0, h], K[0, 0], V[0, 0])
        assert np.abs(res["O"][0, h] - ex).max() <= 1e-9
