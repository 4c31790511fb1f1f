"""The weights X = [V_S, w] (Alg 2 "Compress values") against the oracle's, as an intermediate
("restore a measured X bound"): the fp32 path computes A3 in fp32 on CUDA cores, the bf16
path rounds P = h~(K_S, K) to bf16 for the tensor cores (DESIGN.md error budget); both solve in fp64.
Bounds are the measured maxima (printed with -s) times a ~4x margin, relative to max |X_oracle|."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

try:
    from wc_harness import qkv
except Exception:  # pragma: no cover
    pass

# (dtype, family, shape, r): measured max relative X error on B200 -> bound
CASES = [
    ("f32", "G", (1, 1, 1, 256, 256, 16), 16, 2e-6),
    ("f32", "C", (1, 2, 1, 64, 3000, 64), 48, 2e-5),
    ("bf16", "G", (1, 1, 1, 64, 4096, 128), 128, 4e-3),
    ("bf16", "C", (2, 4, 2, 100, 700, 64), 40, 1e-2),
]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import oracle

    oracle.build()


@pytest.mark.parametrize("dtype,family,shape,r,bound", CASES)
def test_x_against_oracle(dtype, family, shape, r, bound):
    import oracle
    import paper_2602_10056_b200 as wc

    Q, K, V = qkv(*shape, dtype, family, seed=5)
    dev = torch.device("cuda:0")
    sel = wc.select(Q.to(dev), K.to(dev), r, seed=5, block=16)
    cache = wc.weights(K.to(dev), V.to(dev), sel)
    torch.cuda.synchronize()
    res = oracle.forward(Q.double().numpy(), K.double().numpy(), V.double().numpy(), r, seed=5, block=16)
    assert np.array_equal(sel.S.cpu().numpy(), res["S"])
    X = cache.X.cpu().numpy().astype(np.float64)
    rel = np.abs(X - res["X"]).max() / np.abs(res["X"]).max()
    print(f"X rel err {dtype} {family} r={r}: {rel:.3e} (bound {bound:.0e})")
    assert rel <= bound, rel
