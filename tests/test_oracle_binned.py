"""Pins for the binned oracle (Alg 2 CompressKV with B bins; readings Z12, Z13, Z23).

Checked against things other than the binned code itself:
  * B = 1 is the unbinned Alg 4 oracle bit for bit;
  * full-rank bins (r_b = n_b) make every bin's Nystrom weights exact, so WildCat reproduces exact
    softmax attention over ALL keys (Prop.) -- this pins the global recentring, the
    concatenation of the bin coresets and the per-bin value compression at once;
  * bins whose keys repeat m distinct vectors exhaust at r_eff_b = m and are again exact;
  * structural consistency (SPEC "binning consistency"): each bin's pivots are the single-bin RPNys
    on the bin slice with the global kbar, tau_b from the bin's radius and n_b, and stream u*B + b;
  * tau_b from the bin's own radius R_K^b (numpy max norm) and n_b;
  * B not dividing n (Z13): bins of floor(n/B) keys, the last one also holding the remainder -- the
    same per-bin pins hold with the last bin's own size.
"""
import numpy as np
import pytest

from paper_2602_10056_b200.inputs import make_qkv


def _qkv(batch, hq, hkv, m, n, d, family="G", seed=0, distinct=None):
    Q, K, V = make_qkv(batch, hq, hkv, m, n, d, "f32", family, seed, distinct)
    return Q.double().numpy(), K.double().numpy(), V.double().numpy()


@pytest.mark.parametrize("block", [1, 8])
def test_one_bin_is_unbinned(orc, block):
    Q, K, V = _qkv(2, 4, 2, 40, 120, 16, "C", seed=3)
    a = orc.forward(Q, K, V, 20, seed=3, block=block)
    b = orc.forward_binned(Q, K, V, 20, 1, seed=3, block=block)
    assert np.array_equal(a["S"], b["S"]) and np.array_equal(a["r_eff"], b["r_eff"])
    assert np.array_equal(a["O"], b["O"]) and np.array_equal(a["X"], b["X"])
    assert np.allclose(b["stats"][:, 0, :], a["stats"], rtol=0, atol=0)


@pytest.mark.parametrize("bins", [2, 4, 8])
def test_full_rank_bins_are_exact_attention(orc, bins):
    Q, K, V = _qkv(1, 2, 1, 30, 64, 8, "G", seed=5)
    res = orc.forward_binned(Q, K, V, 64, bins, seed=5, clip=False)
    assert res["r_eff"][0] == 64
    ex = np.stack([orc.exact_attention(Q[0, h], K[0, 0], V[0, 0]) for h in range(2)])
    err = np.abs(res["O"][0] - ex).max() / np.abs(V).max()
    assert err < 1e-8, err


def test_distinct_key_bins_exhaust_and_are_exact(orc):
    # every bin repeats 5 distinct key vectors: r_eff_b = 5 per bin, exact attention overall
    bins, nb, d = 4, 40, 8
    rng = np.random.Generator(np.random.PCG64(11))
    K = np.concatenate([rng.standard_normal((5, d))[rng.integers(0, 5, nb)] for _ in range(bins)])[None, None]
    V = rng.standard_normal((1, 1, bins * nb, d))
    Q = rng.standard_normal((1, 1, 25, d))
    res = orc.forward_binned(Q, K, V, 40, bins, seed=11, clip=False)
    assert res["r_eff"][0] == 5 * bins
    ex = orc.exact_attention(Q[0, 0], K[0, 0], V[0, 0])
    assert np.abs(res["O"][0, 0] - ex).max() / np.abs(V).max() < 1e-8


@pytest.mark.parametrize("n", [240, 253])
@pytest.mark.parametrize("block", [1, 4])
def test_bin_pivots_are_single_bin_rpnys(orc, block, n):
    # n = 253 = 4 * 63 + 1: bins of 63, 63, 63 and 64 keys (the remainder in the last bin, Z13)
    Q, K, V = _qkv(1, 2, 1, 50, n, 16, "L", seed=7)
    bins, r = 4, 30
    res = orc.forward_binned(Q, K, V, r, bins, seed=7, block=block)
    rb, R = orc.bin_rank(n, r, bins)
    nb = n // bins
    K64 = K[0, 0]
    kbar, st = orc.prologue(K64, Q[0].reshape(-1, 16))
    tot = 0
    for b in range(bins):
        hi = n if b == bins - 1 else (b + 1) * nb
        Kb = K64[b * nb:hi]
        rk = np.sqrt(((Kb - kbar) ** 2).sum(1).max())
        tau = orc.temperature(1 / np.sqrt(16), st["rq"], rk, hi - b * nb)
        g = (1 / np.sqrt(16)) / tau ** 2
        assert np.isclose(res["stats"][0, b, 3], rk, rtol=1e-13) and np.isclose(res["stats"][0, b, 0], tau, rtol=1e-13)
        if block > 1:
            sel = orc.select_blocked(Kb, kbar, g, g * rk * rk, rb, block, seed=7, unit=b)
        else:
            sel = orc.select(Kb, kbar, g, g * rk * rk, rb, seed=7, unit=b)
        re = sel["r_eff"]
        assert np.array_equal(res["S"][0, tot:tot + re], sel["S"][:re] + b * nb)
        tot += re
    assert res["r_eff"][0] == tot and np.all(res["S"][0, tot:] == -1)


def test_remainder_bin_distinct_keys_exact(orc):
    # bins of 40, 40, 40 and 43 keys (n = 163, B = 4), each repeating 5 distinct vectors: r_eff_b = 5
    # in every bin, the last included, and the binned WildCat is exact attention over all keys
    bins, d, n = 4, 8, 163
    nb = n // bins
    rng = np.random.Generator(np.random.PCG64(13))
    sizes = [nb] * (bins - 1) + [n - (bins - 1) * nb]
    K = np.concatenate([rng.standard_normal((5, d))[rng.integers(0, 5, sz)] for sz in sizes])[None, None]
    V = rng.standard_normal((1, 1, n, d))
    Q = rng.standard_normal((1, 1, 25, d))
    res = orc.forward_binned(Q, K, V, 40, bins, seed=13, clip=False)
    assert res["r_eff"][0] == 5 * bins
    ex = orc.exact_attention(Q[0, 0], K[0, 0], V[0, 0])
    assert np.abs(res["O"][0, 0] - ex).max() / np.abs(V).max() < 1e-8


def test_bins_limits(orc):
    Q, K, V = _qkv(1, 1, 1, 10, 50, 8, seed=1)
    orc.forward_binned(Q, K, V, 12, 3, seed=1)  # 3 does not divide 50: bins of 16, 16 and 18 keys
    with pytest.raises(RuntimeError):
        orc.forward_binned(Q, K, V, 60, 51, seed=1)  # more bins than keys
