"""GPU parity of the options of wc_opts (include/wildcat.h): the PAR2 unit offset,
WC_TAU_ONE / WC_NO_RECENTER and WC_CHECK_FINITE.

Bars as everywhere: pivots bit-exact vs the fp64 oracle run with the same option, outputs within
1e-4 (fp32) / 2e-2 (bf16) of ||V||_max."""
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


@pytest.mark.parametrize("block,bins", [(1, 1), (16, 1), (16, 4), (1, 4)])
def test_unit_offset_partition_bitwise(block, bins):
    """Units [4, 8) run alone with unit_offset = 4 give the full 8-unit run's pivots and outputs bit for
    bit (PAR2: a GPU holding a contiguous unit range of the batch), and match the oracle."""
    Q, K, V = qkv(4, 4, 2, 64, 512, 32, "bf16", "C", seed=21)
    Of, Sf, Rf = run_gpu(Q, K, V, 24, seed=3, block=block, bins=bins)
    Op, Sp, Rp = run_gpu(Q[2:], K[2:], V[2:], 24, seed=3, block=block, bins=bins, unit_offset=4)
    assert np.array_equal(Sf[4:], Sp) and np.array_equal(Rf[4:], Rp)
    assert np.array_equal(Of[2:], Op)
    compare(Q[2:], K[2:], V[2:], 24, "bf16", seed=3, block=block, bins=bins, unit_offset=4)


@pytest.mark.parametrize("tau_one,recenter,family", [(True, True, "L"), (False, False, "G"), (True, False, "C")])
@pytest.mark.parametrize("block", [1, 16])
def test_prologue_options_parity(tau_one, recenter, family, block):
    # WC_NO_RECENTER is tested on near-zero-mean keys: on the L family (per-channel offsets ~3 sigma, x8
    # outliers) the uncentred kernel spans exp(-2 mstar) with mstar in the hundreds, below the fp32
    # exponent range of the A3 / A5 tensor-core epilogues (include/wildcat.h, WC_NO_RECENTER)
    Q, K, V = qkv(2, 4, 2, 100, 1500, 64, "bf16", family, seed=7)
    compare(Q, K, V, 40, "bf16", seed=7, block=block, tau_one=tau_one, recenter=recenter)


@pytest.mark.parametrize("tau_one,recenter", [(True, True), (False, False)])
def test_prologue_options_fp32_binned(tau_one, recenter):
    Q, K, V = qkv(1, 2, 1, 256, 256, 16, "f32", "G", seed=4)
    compare(Q, K, V, 16, "f32", seed=4, bins=4, block=8, tau_one=tau_one, recenter=recenter)
    compare(Q, K, V, 16, "f32", seed=4, tau_one=tau_one, recenter=recenter)


def test_stats_reflect_options():
    import paper_2602_10056_b200 as wc

    Q, K, V = qkv(1, 1, 1, 64, 300, 32, "f32", "L", seed=2)
    dev = torch.device("cuda:0")
    sel = wc.select(Q.to(dev), K.to(dev), 8, tau_one=True, recenter=False)
    st = sel.stats.cpu().numpy()[0]
    beta = 1.0 / np.sqrt(32)
    assert st[0] == 1.0 and st[1] == beta  # tau, g
    assert np.all(st[16:] == 0.0)          # kbar
    rk = np.linalg.norm(K[0, 0].double().numpy(), axis=1).max()
    assert st[3] == pytest.approx(rk, rel=1e-13)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("where", ["Q", "K", "V"])
def test_check_finite(dtype, where):
    import paper_2602_10056_b200 as wc

    dev = torch.device("cuda:0")
    Q, K, V = (x.to(dev) for x in qkv(1, 2, 1, 33, 301, 64, dtype, "G", seed=1))
    O0 = wc.forward(Q, K, V, 16, seed=1)
    O1 = wc.forward(Q, K, V, 16, seed=1, check_finite=True)  # clean inputs: same result
    assert torch.equal(O0, O1)
    bad = {"Q": Q, "K": K, "V": V}[where].clone()
    bad.view(-1)[-1] = float("inf") if where == "V" else float("nan")  # the last element (tail path)
    args = {"Q": Q, "K": K, "V": V}
    args[where] = bad
    with pytest.raises(wc.NonFiniteInput):
        wc.forward(args["Q"], args["K"], args["V"], 16, seed=1, check_finite=True)
    bad.view(-1)[-1] = 0.0
    bad.view(-1)[bad.numel() // 2] = float("-inf")
    args[where] = bad
    with pytest.raises(wc.NonFiniteInput):
        wc.forward(args["Q"], args["K"], args["V"], 16, seed=1, check_finite=True)
