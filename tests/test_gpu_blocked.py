"""GPU parity of the blocked (accelerated) RPCholesky selection (opts.block = b >= 2, reading Z22)
against the fp64 oracle of the same procedure (oracle wco_select_blocked): accepted pivot sequence
bit-exact, r_eff equal, and outputs within the north-star bars (1e-4 fp32, 2e-2 bf16 of ||V||_max).
Sizes span several super-tiles, many co-resident CTAs per unit, ragged tails and exhaustion."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

try:
    from wc_harness import compare, qkv, run_gpu
except Exception:  # pragma: no cover
    pass


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import oracle

    oracle.build()


@pytest.mark.parametrize("block", [2, 8, 16, 20, 32])
def test_cfg1_fp32_blocked(block):
    Q, K, V = qkv(1, 1, 1, 256, 256, 16, "f32", "G", seed=0)
    compare(Q, K, V, 16, "f32", seed=0, block=block)


@pytest.mark.parametrize("family", ["C", "L"])
def test_cfg1_families_blocked(family):
    Q, K, V = qkv(1, 1, 1, 256, 256, 16, "f32", family, seed=3)
    compare(Q, K, V, 16, "f32", seed=3, block=8)


@pytest.mark.parametrize("block", [8, 32])
def test_vit_blocked(block):
    Q, K, V = qkv(64, 12, 12, 197, 197, 64, "bf16", "C", seed=0)
    compare(Q, K, V, 32, "bf16", seed=0, block=block)


@pytest.mark.parametrize("block", [16, 32])
def test_diffusion_shape_blocked(block):
    Q, K, V = qkv(2, 16, 16, 4096, 4096, 64, "bf16", "C", seed=0)
    compare(Q, K, V, 128, "bf16", seed=0, block=block)


@pytest.mark.parametrize("block", [16, 32])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_ragged_gqa_blocked(dtype, block):
    Q, K, V = qkv(2, 8, 2, 77, 1000, 32, dtype, "G", seed=5)
    compare(Q, K, V, 50, dtype, seed=5, block=block)


@pytest.mark.parametrize("block", [16, 25, 32])
def test_multi_cta_unit_blocked(block):
    Q, K, V = qkv(1, 1, 1, 300, 20011, 64, "bf16", "G", seed=9)
    compare(Q, K, V, 64, "bf16", seed=9, block=block)


@pytest.mark.parametrize("block", [16, 32])
def test_fp32_d128_blocked(block):
    # fp32 keys with d = 128: the K row is read in two register chunks
    Q, K, V = qkv(1, 2, 1, 100, 3000, 128, "f32", "G", seed=13)
    compare(Q, K, V, 40, "f32", seed=13, block=block)


@pytest.mark.parametrize("block", [16, 32])
def test_llm_like_blocked(block):
    Q, K, V = qkv(1, 4, 2, 64, 4096, 128, "bf16", "L", seed=2)
    compare(Q, K, V, 96, "bf16", seed=2, block=block)


@pytest.mark.parametrize("r,block", [(512, 16), (1024, 16), (300, 32)])
def test_large_r_blocked(r, block):
    Q, K, V = qkv(1, 2, 1, 200, 6000, 128, "bf16", "G", seed=11)
    compare(Q, K, V, r, "bf16", seed=11, block=block)


@pytest.mark.parametrize("block", [8, 32])
def test_exhaustion_blocked(block):
    Q, K, V = qkv(1, 1, 1, 64, 500, 32, "f32", "D", seed=4, distinct=7)
    out = compare(Q, K, V, 20, "f32", seed=4, block=block)
    assert out["r_eff"][0] == 7
    assert np.all(out["S"][0, 7:] == -1)


@pytest.mark.parametrize("block", [16, 32])
def test_block_stats_and_determinism(block):
    import paper_2602_10056_b200 as wc
    import oracle

    Q, K, V = qkv(1, 2, 2, 50, 5000, 64, "bf16", "G", seed=21)
    dev = torch.device("cuda:0")
    Qd, Kd = Q.to(dev), K.to(dev)
    s1 = wc.select(Qd, Kd, 100, seed=21, block=block)
    s2 = wc.select(Qd, Kd, 100, seed=21, block=block)
    torch.cuda.synchronize()
    assert torch.equal(s1.S, s2.S) and torch.equal(s1.L, s2.L)
    st = s1.stats.cpu().numpy()
    for u in range(2):
        K64 = K[0, u].double().numpy()
        kbar, ost = oracle.prologue(K64, Q[0, u].double().numpy())
        ref = oracle.select_blocked(K64, kbar, ost["g"], ost["mstar"], 100, block, seed=21, unit=u)
        assert np.array_equal(s1.S.cpu().numpy()[u], ref["S"])
        assert int(st[u, 6]) == ref["nblocks"] and int(st[u, 7]) == ref["ncand"]
        # L = F[:, S] (lower-triangular Cholesky factor of h~(K_S, K_S)) against the oracle's
        Lg = s1.L.cpu().numpy()[u]
        assert np.abs(Lg - ref["L"]).max() <= 1e-9 * np.abs(ref["L"]).max()


@pytest.mark.slow
@pytest.mark.parametrize("block", [16, 32])
def test_headline_full_size_blocked(block):
    """The bench's headline (n = m = 65536, d = 128, r = 256, bf16, seed 0) in the launch
    configuration bench.py times (blocked selection): pivots bit-exact against the oracle's
    wco_select_blocked, and the outputs of 1024 sampled query rows against the oracle's weights and
    attend (Alg 2 + Alg 3 over all n keys) within the bf16 bar."""
    import paper_2602_10056_b200 as wc
    import oracle
    from paper_2602_10056_b200.inputs import make_config, CONFIGS, query_sample

    Q, K, V = make_config(CONFIGS["headline"])
    dev = torch.device("cuda:0")
    S = torch.empty(1, 256, dtype=torch.int32, device=dev)
    R = torch.empty(1, dtype=torch.int32, device=dev)
    O = wc.forward(Q.to(dev), K.to(dev), V.to(dev), 256, seed=0, block=block, S=S, r_eff=R)
    torch.cuda.synchronize()
    K64, V64 = K[0, 0].double().numpy(), V[0, 0].double().numpy()
    kbar, st = oracle.prologue(K64, Q[0, 0].double().numpy())
    ref = oracle.select_blocked(K64, kbar, st["g"], st["mstar"], 256, block, seed=0, unit=0)
    assert np.array_equal(S.cpu().numpy()[0], ref["S"]) and int(R.cpu()[0]) == ref["r_eff"]
    re = ref["r_eff"]
    X = oracle.weights(K64, V64, ref["S"], re, kbar, st["g"], st["mstar"])
    rows = query_sample(65536, 1024, seed=7)
    Or = oracle.attend(Q[0, 0].double().numpy()[rows], K64[ref["S"][:re]], X[:re], re, 1.0 / np.sqrt(128),
                       V64.min(0), V64.max(0))
    err = np.abs(O[0, 0].cpu().double().numpy()[rows] - Or).max() / np.abs(V64).max()
    assert err <= 2e-2, err
