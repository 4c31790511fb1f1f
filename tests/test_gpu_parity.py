"""GPU (CUDA path via the C ABI) vs fp64 oracle parity, element by element.

Bars (BASELINE.json north star): pivot indices bit-exact, r_eff equal, and
max |O_gpu - O_oracle| / ||V||_max <= 1e-4 (fp32 inputs) or 2e-2 (bf16 inputs).
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

try:
    from wc_harness import compare, qkv, run_gpu, run_oracle
except Exception:  # pragma: no cover
    pass


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import oracle

    oracle.build()


def test_cfg1_fp32():
    # BASELINE.json configs[0]: single head n=256, d=16, r=16, fp32, seed 0
    Q, K, V = qkv(1, 1, 1, 256, 256, 16, "f32", "G", seed=0)
    out = compare(Q, K, V, 16, "f32", seed=0)
    assert out["r_eff"][0] == 16


@pytest.mark.parametrize("family", ["G", "C", "L"])
def test_cfg1_families_fp32(family):
    Q, K, V = qkv(1, 1, 1, 256, 256, 16, "f32", family, seed=3)
    compare(Q, K, V, 16, "f32", seed=3)


def test_vit_bf16():
    # configs[1]: ViT-B/16, batch 64, 12 heads, n = 197, d = 64, r = 32, bf16
    Q, K, V = qkv(64, 12, 12, 197, 197, 64, "bf16", "C", seed=0)
    compare(Q, K, V, 32, "bf16", seed=0)


def test_diffusion_shape_bf16():
    # configs[2] shape (n = 4096, d = 64, r = 128) on 2 of the 8 batches (32 units)
    Q, K, V = qkv(2, 16, 16, 4096, 4096, 64, "bf16", "C", seed=0)
    compare(Q, K, V, 128, "bf16", seed=0)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_ragged_gqa(dtype):
    # ragged n and m (not multiples of any tile), GQA 4 q-heads per kv-head, 2 batches
    Q, K, V = qkv(2, 8, 2, 77, 1000, 32, dtype, "G", seed=5)
    compare(Q, K, V, 50, dtype, seed=5)


def test_multi_cta_unit():
    # one unit large enough to be split over many co-resident CTAs (grid-group barrier path)
    Q, K, V = qkv(1, 1, 1, 300, 20011, 64, "bf16", "G", seed=9)
    compare(Q, K, V, 64, "bf16", seed=9)


def test_llm_like_conditioning():
    # LLM-like keys (offsets + outlier channels): ill-conditioned coreset kernel
    Q, K, V = qkv(1, 4, 2, 64, 4096, 128, "bf16", "L", seed=2)
    compare(Q, K, V, 96, "bf16", seed=2)


@pytest.mark.parametrize("d,r,family", [(128, 512, "G"), (64, 320, "L"), (128, 1024, "C")])
def test_large_r_streamed_attend(d, r, family):
    # r > 256: the tcgen05 attend streams the coreset in 128-row chunks with lazy max rescaling
    # (LLM-like keys make later chunks raise the running max); r = 320 leaves a ragged last chunk
    Q, K, V = qkv(1, 4, 2, 300, 3000, d, "bf16", family, seed=11)
    compare(Q, K, V, r, "bf16", seed=11)


def test_large_r_exhausted():
    # r_eff (distinct keys) far below r: fewer chunks than r / 128, zero-padded tail
    Q, K, V = qkv(1, 2, 1, 200, 2000, 128, "bf16", "D", seed=6, distinct=150)
    out = compare(Q, K, V, 512, "bf16", seed=6)
    assert out["r_eff"][0] == 150


def test_rank_one_and_full_rank():
    Q, K, V = qkv(1, 1, 1, 40, 64, 16, "f32", "G", seed=1)
    compare(Q, K, V, 1, "f32", seed=1)
    out = compare(Q, K, V, 64, "f32", seed=1)
    import oracle

    # r = n: exact attention (up to exhaustion)
    ex = oracle.exact_attention(Q[0, 0].double().numpy(), K[0, 0].double().numpy(), V[0, 0].double().numpy())
    assert np.abs(out["O"][0, 0] - ex).max() <= 1e-3 * np.abs(V.double().numpy()).max()


def test_distinct_keys_exhaustion():
    Q, K, V = qkv(1, 1, 1, 64, 500, 32, "f32", "D", seed=4, distinct=7)
    out = compare(Q, K, V, 20, "f32", seed=4)
    assert out["r_eff"][0] == 7
    assert np.all(out["S"][0, 7:] == -1)


def test_single_key_and_empty_queries():
    Q, K, V = qkv(1, 1, 1, 5, 1, 16, "f32", "G", seed=0)
    compare(Q, K, V, 1, "f32")
    Q0 = Q[:, :, :0]
    O, S, R = run_gpu(Q0, K, V, 1)
    assert O.shape == (1, 1, 0, 16) and R[0] == 1


def test_split_api_equals_forward_and_is_deterministic():
    import paper_2602_10056_b200 as wc

    Q, K, V = qkv(2, 4, 2, 100, 700, 64, "bf16", "C", seed=8)
    dev = torch.device("cuda:0")
    Qd, Kd, Vd = Q.to(dev), K.to(dev), V.to(dev)
    O1 = wc.forward(Qd, Kd, Vd, 40, seed=8)
    O2 = wc.forward(Qd, Kd, Vd, 40, seed=8)
    sel = wc.select(Qd, Kd, 40, seed=8)
    cache = wc.weights(Kd, Vd, sel)
    O3 = wc.attend(Qd, cache)
    torch.cuda.synchronize()
    assert torch.equal(O1, O2)
    assert torch.equal(O1, O3)
    # selection outputs against the oracle: stats, L, X
    import oracle

    res = oracle.forward(Q.double().numpy(), K.double().numpy(), V.double().numpy(), 40, seed=8)
    assert np.array_equal(sel.S.cpu().numpy(), res["S"])
    st = sel.stats.cpu().numpy()
    assert np.allclose(st[:, :5], res["stats"], rtol=1e-12, atol=0)
    # X = [V_S, w]: the bf16 path rounds P = h~(K_S, K) to bf16 in the A3 GEMM (error
    # budget), so X carries ~2^-9-relative noise amplified by cond(h~(K_S,K_S)); the output bar
    # (2e-2 of ||V||_max) is checked by the other tests.
    X = cache.X.cpu().numpy().astype(np.float64)
    rel = np.abs(X - res["X"]).max() / np.abs(res["X"]).max()
    assert rel < 2e-2, rel


@pytest.mark.slow
def test_headline_full_size_pivots_and_sampled_outputs():
    # configs as timed by bench.py: 1 unit, n = m = 65536, d = 128, r = 256, bf16
    import oracle
    import paper_2602_10056_b200 as wc
    from paper_2602_10056_b200.inputs import query_sample

    Q, K, V = qkv(1, 1, 1, 65536, 65536, 128, "bf16", "G", seed=0)
    dev = torch.device("cuda:0")
    Kd, Vd, Qd = K.to(dev), V.to(dev), Q.to(dev)
    S = torch.empty(1, 256, dtype=torch.int32, device=dev)
    R = torch.empty(1, dtype=torch.int32, device=dev)
    O = wc.forward(Qd, Kd, Vd, 256, seed=0, S=S, r_eff=R).float().cpu().numpy()
    K64, V64, Q64 = K[0, 0].double().numpy(), V[0, 0].double().numpy(), Q[0, 0].double().numpy()
    kbar, st = oracle.prologue(K64, Q64)
    sel = oracle.select(K64, kbar, st["g"], st["mstar"], 256, seed=0, unit=0)
    assert np.array_equal(S.cpu().numpy()[0], sel["S"]) and int(R.cpu()[0]) == sel["r_eff"]
    X = oracle.weights(K64, V64, sel["S"], sel["r_eff"], kbar, st["g"], st["mstar"])
    rows = query_sample(65536, 2048)
    Oo = oracle.attend(Q64[rows], K64[sel["S"]], X, sel["r_eff"], 1 / math.sqrt(128), V64.min(0), V64.max(0))
    err = np.abs(O[0, 0][rows] - Oo).max() / np.abs(V64).max()
    assert err <= 2e-2, err


@pytest.mark.parametrize("block", [1, 16])
def test_forward_host_matches_device_forward(block):
    # the end-to-end host-buffer path (split C-ABI calls, V copied on a side stream) == wildcat_forward
    import paper_2602_10056_b200 as wc

    Q, K, V = qkv(2, 4, 2, 300, 3000, 64, "bf16", "C", seed=12)
    dev = torch.device("cuda:0")
    Od = wc.forward(Q.to(dev), K.to(dev), V.to(dev), 64, seed=12, block=block)
    torch.cuda.synchronize()
    Qh, Kh, Vh = (x.pin_memory() for x in (Q, K, V))
    for _ in range(2):  # second call reuses the cached device buffers
        Oh = wc.forward_host(Qh, Kh, Vh, 64, seed=12, block=block)
        assert torch.equal(Oh, Od.cpu())


@pytest.mark.gpu
@pytest.mark.parametrize("block", [1, 16])
def test_host_pipeline_matches_device_forward(block):
    # streamed host batches (HostPipeline: H2D / forward / D2H on three event-ordered streams, two
    # device slots reused every other step) == wildcat_forward on each batch, bit for bit
    import paper_2602_10056_b200 as wc

    dev = torch.device("cuda:0")
    batches = [qkv(2, 4, 2, 300, 3000, 64, "bf16", "C", seed=20 + k) for k in range(5)]
    want = []
    for Q, K, V in batches:
        want.append(wc.forward(Q.to(dev), K.to(dev), V.to(dev), 64, seed=12, block=block).cpu())
    Q0, K0, _ = batches[0]
    pipe = wc.HostPipeline(Q0, K0, 64, seed=12, block=block)
    pinned = [tuple(x.pin_memory() for x in b) for b in batches]
    outs = [torch.empty(Q0.shape, dtype=Q0.dtype, pin_memory=True) for _ in batches]
    for (Qh, Kh, Vh), Oh in zip(pinned, outs):
        pipe.submit(Qh, Kh, Vh, Oh)
    pipe.synchronize()
    for k, Oh in enumerate(outs):
        assert torch.equal(Oh, want[k]), k
    with pytest.raises(wc.WildcatError):
        pipe.submit(Q0.to(dev), K0, K0, outs[0])


@pytest.mark.gpu
def test_binding_rejects_mismatched_tensors():
    import paper_2602_10056_b200 as wc
    # the C ABI takes raw pointers, so the wrappers must refuse tensors that disagree
    # with the shape (dtype, batch / d, sizes of S / r_eff / out) before any launch
    dev = torch.device("cuda:0")
    Q, K, V = (x.to(dev) for x in qkv(1, 2, 1, 64, 128, 64, "bf16"))
    with pytest.raises(wc.WildcatError, match="dtype"):
        wc.forward(Q.float(), K, V, 8)
    with pytest.raises(wc.WildcatError, match="elements"):
        wc.forward(torch.cat([Q, Q]), K, V, 8)  # Q batch larger than K's
    with pytest.raises(wc.WildcatError, match="elements"):
        wc.forward(Q, K, V[:, :, :100].contiguous(), 8)
    with pytest.raises(wc.WildcatError, match="S"):
        wc.forward(Q, K, V, 8, S=torch.empty(1, 4, dtype=torch.int32, device=dev))
    with pytest.raises(wc.WildcatError, match="contiguous"):
        B = wc._binding
        sh = B.make_shape(Q, K, 8)
        B.wildcat_forward(sh, B.make_opts(), Q, K, V, torch.empty_like(Q).transpose(2, 3), None, None,
                          wc._workspace(sh, B.WC_OP_FORWARD, dev))
    sel = wc.select(Q, K, 8)
    cache = wc.weights(K, V, sel)
    with pytest.raises(wc.WildcatError, match="dtype"):
        wc.attend(Q.float(), cache)
    # a correct call still runs
    O = wc.forward(Q, K, V, 8)
    torch.cuda.synchronize()
    assert torch.isfinite(O.float()).all()
