"""GPU parity of Alg 2 binning (shape.bins = B > 1; readings Z12, Z13, Z23) against the binned
fp64 oracle (wco_forward_binned): the concatenated pivots bit-exact, r_eff equal, outputs within
the north-star bars.  Sequential and blocked selection, fp32 and bf16, GQA, capped bin ranks."""
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


@pytest.mark.parametrize("bins,block", [(2, 1), (4, 1), (4, 8)])
def test_binned_fp32(bins, block):
    Q, K, V = qkv(1, 2, 1, 256, 256, 16, "f32", "G", seed=0)
    compare(Q, K, V, 32, "f32", seed=0, bins=bins, block=block)


@pytest.mark.parametrize("block", [1, 16])
def test_binned_diffusion_shape(block):
    # configs[2] shape (n = 4096, d = 64, r = 128) with B = 8 bins (r_b = 16), 2 x 4 units
    Q, K, V = qkv(2, 4, 4, 4096, 4096, 64, "bf16", "C", seed=1)
    compare(Q, K, V, 128, "bf16", seed=1, bins=8, block=block)


def test_binned_gqa_ragged_rank():
    # r not divisible by B: r_b = ceil(r/B) (R = B r_b > r), ragged m, GQA 4:1
    Q, K, V = qkv(2, 8, 2, 77, 1200, 32, "bf16", "L", seed=4)
    out = compare(Q, K, V, 50, "bf16", seed=4, bins=3)
    assert out["S"].shape[1] == 3 * 17


def test_full_rank_bins_exact_attention():
    import oracle

    Q, K, V = qkv(1, 2, 1, 40, 64, 16, "f32", "G", seed=2)
    out = compare(Q, K, V, 64, "f32", seed=2, bins=8, clip=False)
    ex = np.stack([oracle.exact_attention(Q[0, h].double().numpy(), K[0, 0].double().numpy(),
                                          V[0, 0].double().numpy()) for h in range(2)])
    assert np.abs(out["O"][0] - ex).max() <= 1e-4 * np.abs(V.double().numpy()).max()


def test_binned_split_api_equals_forward():
    import paper_2602_10056_b200 as wc

    Q, K, V = qkv(2, 4, 2, 100, 2048, 64, "bf16", "C", seed=8)
    dev = torch.device("cuda:0")
    Qd, Kd, Vd = Q.to(dev), K.to(dev), V.to(dev)
    O1 = wc.forward(Qd, Kd, Vd, 64, seed=8, bins=4, block=8)
    sel = wc.select(Qd, Kd, 64, seed=8, bins=4, block=8)
    cache = wc.weights(Kd, Vd, sel)
    O2 = wc.attend(Qd, cache)
    torch.cuda.synchronize()
    assert torch.equal(O1, O2)
    st = sel.stats.cpu().numpy()
    import oracle

    res = oracle.forward_binned(Q.double().numpy(), K.double().numpy(), V.double().numpy(), 64, 4, seed=8, block=8)
    assert np.array_equal(sel.S.cpu().numpy(), res["S"])
    assert np.allclose(st[:, :5], res["stats"].reshape(-1, 5), rtol=1e-12, atol=0)


@pytest.mark.parametrize("n,bins,block,dtype,d", [(50, 3, 1, "f32", 16), (50, 3, 4, "f32", 16),
                                                  (4099, 8, 16, "bf16", 64), (1203, 7, 1, "bf16", 32),
                                                  (20011, 16, 16, "bf16", 128)])
def test_remainder_bin(n, bins, block, dtype, d):
    """B not dividing n (reading Z13): bins of floor(n/B) keys, the last one also holding the
    remainder -- pivots bit-exact and outputs within the bar against the oracle's wco_forward_binned."""
    Q, K, V = qkv(2, 4, 2, 60, n, d, dtype, "C", seed=13)
    compare(Q, K, V, 6 * bins, dtype, seed=13, bins=bins, block=block)


def test_remainder_bin_split_api_and_kv():
    import paper_2602_10056_b200 as wc
    import oracle

    # split API with a remainder (select -> weights unpacks the bins of S, the last one holding the
    # remainder), and the KV cache with a middle that 7 bins do not divide
    Q, K, V = qkv(1, 4, 2, 64, 1000, 64, "bf16", "L", seed=21)
    dev = torch.device("cuda:0")
    Qd, Kd, Vd = Q.to(dev), K.to(dev), V.to(dev)
    O1 = wc.forward(Qd, Kd, Vd, 42, seed=21, bins=7, block=8)
    sel = wc.select(Qd, Kd, 42, seed=21, bins=7, block=8)
    O2 = wc.attend(Qd, wc.weights(Kd, Vd, sel))
    torch.cuda.synchronize()
    assert torch.equal(O1, O2)
    res = oracle.forward_binned(Q.double().numpy(), K.double().numpy(), V.double().numpy(), 42, 7, seed=21, block=8)
    assert np.array_equal(sel.S.cpu().numpy(), res["S"])
    cache = wc.compress_kv(Qd, Kd, Vd, 42, keep_first=32, keep_last=32, bins=7, block=8, seed=21)
    ref = oracle.compress_kv(Q.double().numpy(), K.double().numpy(), V.double().numpy(), 42, keep_first=32, keep_last=32,
                             bins=7, block=8, seed=21)
    assert np.array_equal(cache.r_eff.cpu().numpy(), ref["c_eff"])
