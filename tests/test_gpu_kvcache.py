"""GPU parity of KV-cache compression (wildcat_compress_kv, E3 protocol P:667-669,
reading Z24) and of the decode-shaped WtdAttn (wildcat_attend with m <= 16 queries per q-head)
against the fp64 oracle (wco_compress_kv + wco_attend): coreset token indices bit-exact, the cache's
retained rows and key rows byte-exact, c_eff and the value range exact, decode outputs within the
north-star bars; degenerate splits reduce to exact attention."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

try:
    from wc_harness import TOL, compare, qkv
except Exception:  # pragma: no cover
    pass


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import oracle

    oracle.build()


def _np(t):
    return t.double().cpu().numpy()


def _kv_case(Q, K, V, r, kf, kl, dtype, bins=1, block=1, seed=0, rq=None, Qdec=None, clip=True):
    import oracle
    import paper_2602_10056_b200 as wc

    dev = torch.device("cuda:0")
    Qd, Kd, Vd = Q.to(dev), K.to(dev), V.to(dev)
    units = K.shape[0] * K.shape[1]
    C = wc.kv_capacity(K.shape[2], r, kf, kl, bins)
    R = C - kf - kl
    S = torch.empty(units, max(R, 1), dtype=torch.int32, device=dev)
    cache = wc.compress_kv(Qd, Kd, Vd, r, keep_first=kf, keep_last=kl, bins=bins, block=block, seed=seed, rq=rq,
                           S=S)
    Qn = Q if Qdec is None else Qdec
    Od = wc.attend(Qn.to(dev), cache, clip=clip)
    torch.cuda.synchronize()
    orc = oracle.compress_kv(_np(Q), _np(K), _np(V), r, keep_first=kf, keep_last=kl, bins=bins, seed=seed,
                             rq=-1.0 if rq is None else rq, block=block)
    assert np.array_equal(cache.r_eff.cpu().numpy(), orc["c_eff"])
    assert np.array_equal(S.cpu().numpy()[:, :R], orc["S"])
    assert np.array_equal(_np(cache.KC), orc["KC"])           # key rows are copies
    kept = kf + kl
    assert np.array_equal(_np(cache.VC)[:, :kept], orc["XC"][:, :kept, :-1])  # retained (v_l, 1) rows exact
    assert np.array_equal(_np(cache.WC)[:, :kept], orc["XC"][:, :kept, -1])
    # coreset rows (V_S rounded to the cache dtype, w in fp32) are checked through the decode outputs
    # below: as an intermediate, [V_S, w] carries the conditioning of h~(K_S, K_S) (tests/test_gpu_xweights.py)
    assert np.array_equal(_np(cache.vmin), orc["vmin"]) and np.array_equal(_np(cache.vmax), orc["vmax"])
    Oo = oracle.cache_attend(_np(Qn), orc["KC"], orc["XC"], orc["c_eff"], orc["vmin"], orc["vmax"], K.shape[1],
                             clip=clip)
    err = float(np.abs(_np(Od) - Oo).max()) / float(np.abs(_np(V)).max())
    assert err <= TOL[dtype], f"decode err {err:.3e}"
    return dict(err=err, cache=cache, orc=orc, O=_np(Od))


@pytest.mark.parametrize("kf,kl,bins,block", [(4, 4, 1, 1), (32, 32, 1, 8), (0, 16, 2, 1), (9, 0, 1, 16),
                                              (32, 32, 4, 4)])
def test_compress_kv_fp32(kf, kl, bins, block):
    Q, K, V = qkv(1, 4, 2, 64, 576, 16, "f32", "G", seed=3)
    _kv_case(Q, K, V, 40, kf, kl, "f32", bins=bins, block=block, seed=3)


@pytest.mark.parametrize("m_dec", [1, 3, 16])
def test_compress_kv_bf16_gqa_decode(m_dec):
    # GQA 4:1, d = 128, the prompt's queries define R_Q; decode with m_dec new queries per q-head
    Q, K, V = qkv(2, 8, 2, 256, 2112, 128, "bf16", "L", seed=5)
    Qdec = qkv(2, 8, 2, m_dec, 16, 128, "bf16", "L", seed=99)[0]
    _kv_case(Q, K, V, 128, 32, 32, "bf16", block=16, seed=5, Qdec=Qdec)


def test_compress_kv_large_cache_chunks():
    # r = 512 coreset rows + 64 retained: 9 cache chunks of 64 rows per unit in the decode kernel
    Q, K, V = qkv(1, 4, 1, 128, 4160, 64, "bf16", "C", seed=6)
    Qdec = qkv(1, 4, 1, 1, 16, 64, "bf16", "C", seed=7)[0]
    _kv_case(Q, K, V, 512, 32, 32, "bf16", block=16, seed=6, Qdec=Qdec)


def test_all_retained_is_exact_attention():
    import oracle

    Q, K, V = qkv(1, 2, 1, 5, 96, 32, "f32", "G", seed=8)
    out = _kv_case(Q, K, V, 8, 40, 56, "f32", clip=False)
    assert int(out["cache"].r_eff[0]) == 96
    ex = np.stack([oracle.exact_attention(_np(Q[0, h]), _np(K[0, 0]), _np(V[0, 0])) for h in range(2)])
    assert np.abs(out["O"][0] - ex).max() <= 1e-5 * np.abs(_np(V)).max()


def test_full_rank_middle_is_exact_attention():
    import oracle

    Q, K, V = qkv(1, 2, 1, 7, 128, 16, "f32", "G", seed=9)
    out = _kv_case(Q, K, V, 96, 16, 16, "f32", clip=False)
    ex = np.stack([oracle.exact_attention(_np(Q[0, h]), _np(K[0, 0]), _np(V[0, 0])) for h in range(2)])
    assert np.abs(out["O"][0] - ex).max() <= 1e-4 * np.abs(_np(V)).max()


@pytest.mark.parametrize("m,dtype,d", [(1, "f32", 16), (5, "bf16", 64), (16, "bf16", 128), (2, "f32", 128)])
def test_decode_kernel_in_forward(m, dtype, d):
    # forward with m <= 16 queries per q-head routes A5 through the split-cache decode kernel
    Q, K, V = qkv(2, 4, 2, m, 1000, d, dtype, "G", seed=11)
    compare(Q, K, V, 96, dtype, seed=11, block=8)


def test_invalid_kv_split_rejected():
    import paper_2602_10056_b200 as wc

    Q, K, V = qkv(1, 1, 1, 4, 100, 16, "f32", "G", seed=1)
    dev = torch.device("cuda:0")
    with pytest.raises(wc.WildcatError):
        wc.compress_kv(Q.to(dev), K.to(dev), V.to(dev), 8, keep_first=60, keep_last=60)
    with pytest.raises(wc.WildcatError):
        wc.compress_kv(Q.to(dev), K.to(dev), V.to(dev), 8, keep_first=1, keep_last=0, bins=9)  # more bins than r
    # 2 bins of the 99 middle tokens (49 + 50, reading Z13) are valid
    cache = wc.compress_kv(Q.to(dev), K.to(dev), V.to(dev), 8, keep_first=1, keep_last=0, bins=2)
    assert int(cache.r_eff.cpu()[0]) == 1 + 8


def test_kv_llm32k_full_size():
    """configs[3] shapes (GQA 32/8, n = 32768, d = 128, L family) with the E3 split (32 + 32 retained),
    r = 256, blocked selection: unit 0's coreset bit-exact vs the oracle, its 4 q-heads' decode outputs
    within the bf16 bar, every unit's c_eff = 64 + r."""
    import oracle
    import paper_2602_10056_b200 as wc

    dev = torch.device("cuda:0")
    Q, K, V = qkv(1, 32, 8, 512, 32768, 128, "bf16", "L", seed=0)
    Qdec = qkv(1, 32, 8, 1, 16, 128, "bf16", "L", seed=1)[0]
    S = torch.empty(8, 256, dtype=torch.int32, device=dev)
    cache = wc.compress_kv(Q.to(dev), K.to(dev), V.to(dev), 256, keep_first=32, keep_last=32, block=16, S=S)
    Od = wc.attend(Qdec.to(dev), cache)
    torch.cuda.synchronize()
    assert (cache.r_eff.cpu() == 64 + 256).all()
    orc = oracle.compress_kv(_np(Q[:, :4]), _np(K[:, :1]), _np(V[:, :1]), 256, keep_first=32, keep_last=32,
                             block=16)
    assert np.array_equal(S.cpu().numpy()[0], orc["S"][0])
    Oo = oracle.cache_attend(_np(Qdec[:, :4]), orc["KC"], orc["XC"], orc["c_eff"], orc["vmin"], orc["vmax"], 1)
    err = float(np.abs(_np(Od[:, :4]) - Oo).max()) / float(np.abs(_np(V[:, :1])).max())
    assert err <= TOL["bf16"], err


@pytest.mark.parametrize("d,g,m_dec", [(16, 4, 1), (32, 2, 2), (64, 1, 3), (128, 4, 1)])
def test_decode_token_tensor_core_scores(d, g, m_dec):
    # group * m <= 4: one decode token of a GQA group -> tensor-core scores (QR = 4) for every d
    Q, K, V = qkv(1, 2 * g, 2, 64, 700, d, "bf16", "G", seed=21)
    Qdec = qkv(1, 2 * g, 2, m_dec, 16, d, "bf16", "G", seed=22)[0]
    _kv_case(Q, K, V, 96, 8, 8, "bf16", block=8, seed=21, Qdec=Qdec)
