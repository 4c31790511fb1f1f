"""Pins for the KV-cache compression oracle (wco_compress_kv: P:366-369 prefill compression, the
E3 protocol's retained first/last tokens P:667-669; reading Z24 = the cache is the union of exact
retained entries (k_l, [v_l, 1]) and the CompressKV coreset (k_s, [V_S, w]_s)).

Checked against things other than the KV code itself:
  * nothing compressed (keep_first + keep_last = n): WtdAttn over the cache IS exact softmax
    attention (Eq. 1) over all keys;
  * a full-rank middle (r = n_mid): the Nystrom weights are exact, so the cache again
    reproduces exact attention over ALL n keys -- a dropped retained row, a wrong [v, 1] row, a
    shifted middle slice or a per-part softmax shift fails this;
  * a middle repeating m distinct key vectors exhausts at r_eff = m and is exact;
  * keep_first = keep_last = 0 is the Alg 2/Alg 4 oracle (wco_forward / wco_forward_binned) bit for
    bit; the middle's pivots are those of the forward oracle on the middle slice, shifted;
  * the clip range spans all n values, including the retained rows.
"""
import numpy as np
import pytest

from paper_2602_10056_b200.inputs import make_qkv


def _qkv(batch, hq, hkv, m, n, d, family="G", seed=0, distinct=None):
    Q, K, V = make_qkv(batch, hq, hkv, m, n, d, "f32", family, seed, distinct)
    return Q.double().numpy(), K.double().numpy(), V.double().numpy()


def _exact(orc, Q, K, V):
    batch, hq = Q.shape[:2]
    g = hq // K.shape[1]
    return np.stack([np.stack([orc.exact_attention(Q[b, h], K[b, h // g], V[b, h // g]) for h in range(hq)])
                     for b in range(batch)])


def _attend(orc, Q, c, hkv, clip=True):
    return orc.cache_attend(Q, c["KC"], c["XC"], c["c_eff"], c["vmin"], c["vmax"], hkv, clip=clip)


def test_all_retained_is_exact_attention(orc):
    Q, K, V = _qkv(1, 4, 2, 12, 48, 16, "G", seed=1)
    c = orc.compress_kv(Q, K, V, 8, keep_first=20, keep_last=28)
    assert list(c["c_eff"]) == [48, 48] and c["S"].shape[1] == 0
    err = np.abs(_attend(orc, Q, c, 2, clip=False) - _exact(orc, Q, K, V)).max()
    assert err < 1e-13, err


@pytest.mark.parametrize("kf,kl,bins", [(4, 4, 1), (0, 8, 1), (7, 0, 1), (8, 8, 2), (3, 5, 4)])
def test_full_rank_middle_is_exact_attention(orc, kf, kl, bins):
    n = 72
    Q, K, V = _qkv(2, 4, 2, 10, n, 8, "C", seed=2)
    nmid = n - kf - kl
    c = orc.compress_kv(Q, K, V, nmid, keep_first=kf, keep_last=kl, bins=bins, seed=2)
    assert list(c["c_eff"]) == [n] * 4
    err = np.abs(_attend(orc, Q, c, 2, clip=False) - _exact(orc, Q, K, V)).max() / np.abs(V).max()
    assert err < 1e-8, err


def test_distinct_middle_exhausts_and_is_exact(orc):
    kf, kl, nmid, d = 6, 10, 50, 8
    rng = np.random.Generator(np.random.PCG64(13))
    Kmid = rng.standard_normal((5, d))[rng.integers(0, 5, nmid)]
    K = np.concatenate([rng.standard_normal((kf, d)), Kmid, rng.standard_normal((kl, d))])[None, None]
    V = rng.standard_normal((1, 1, kf + nmid + kl, d))
    Q = rng.standard_normal((1, 2, 9, d))
    c = orc.compress_kv(Q, K, V, 30, keep_first=kf, keep_last=kl, seed=13)
    assert c["c_eff"][0] == kf + kl + 5
    err = np.abs(_attend(orc, Q, c, 1, clip=False) - _exact(orc, Q, K, V)).max() / np.abs(V).max()
    assert err < 1e-8, err


@pytest.mark.parametrize("bins,block", [(1, 1), (1, 8), (4, 1), (2, 4)])
def test_no_retained_tokens_is_the_forward_oracle(orc, bins, block):
    Q, K, V = _qkv(2, 4, 2, 20, 96, 16, "L", seed=4)
    r = 24
    c = orc.compress_kv(Q, K, V, r, bins=bins, block=block, seed=4)
    f = orc.forward(Q, K, V, r, seed=4, bins=bins, block=block)
    assert np.array_equal(c["S"], f["S"]) and np.array_equal(c["c_eff"], f["r_eff"])
    assert np.array_equal(c["XC"], f["X"])
    O = _attend(orc, Q, c, 2)
    assert np.array_equal(O, f["O"])


def test_middle_pivots_are_forward_on_the_slice(orc):
    kf, kl = 16, 32
    Q, K, V = _qkv(1, 2, 2, 8, 240, 16, "G", seed=6)
    rq = 7.5  # fixed R_Q, so the slice forward sees the same temperature input
    c = orc.compress_kv(Q, K, V, 20, keep_first=kf, keep_last=kl, bins=2, seed=6, rq=rq)
    f = orc.forward(Q, K[:, :, kf:-kl], V[:, :, kf:-kl], 20, seed=6, bins=2, rq=rq)
    valid = f["S"] >= 0
    assert np.array_equal(c["S"][valid], f["S"][valid] + kf)
    assert np.all(c["S"][~valid] == -1)
    for u in range(2):
        re = int(f["r_eff"][u])
        KC, XC = c["KC"][u], c["XC"][u]
        kept = np.concatenate([np.arange(kf), np.arange(240 - kl, 240)])
        assert np.array_equal(KC[:kf + kl], K[0, u][kept])
        assert np.array_equal(XC[:kf + kl, :16], V[0, u][kept]) and np.all(XC[:kf + kl, 16] == 1.0)
        assert np.array_equal(KC[kf + kl:kf + kl + re], K[0, u][c["S"][u, :re]])
        assert np.array_equal(XC[kf + kl:kf + kl + re], f["X"][u, :re])
        assert np.all(KC[kf + kl + re:] == 0) and np.all(XC[kf + kl + re:] == 0)


def test_clip_range_spans_retained_values(orc):
    Q, K, V = _qkv(1, 1, 1, 6, 64, 8, "G", seed=8)
    V[0, 0, 1, 3] = 50.0    # a retained first token
    V[0, 0, -2, 5] = -40.0  # a retained last token
    c = orc.compress_kv(Q, K, V, 8, keep_first=4, keep_last=4)
    assert np.array_equal(c["vmin"][0], V[0, 0].min(axis=0))
    assert np.array_equal(c["vmax"][0], V[0, 0].max(axis=0))


def test_invalid_split_raises(orc):
    Q, K, V = _qkv(1, 1, 1, 4, 40, 8)
    with pytest.raises(ValueError):
        orc.compress_kv(Q, K, V, 4, keep_first=30, keep_last=20)
    with pytest.raises(ValueError):
        orc.compress_kv(Q, K, V, 60, keep_first=3, keep_last=0, bins=38)  # 37 middle tokens, 38 bins
    orc.compress_kv(Q, K, V, 8, keep_first=3, keep_last=0, bins=2)  # bins of 18 and 19 (Z13 remainder)
