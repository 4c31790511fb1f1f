"""n-sharded path (PAR3) on the GPU: with a world-size-1 NCCL communicator the sharded protocol
(allgather of rank totals, packet allreduce, Y~ allreduce) must reproduce the oracle's pivots
bit-exactly and its outputs within the bf16 bar.  (Only one GPU is available to the test runs;
the multi-rank protocol itself is checked on CPU by tests/test_nshard_protocol.py.)"""
import math
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["nccl", "p2p"])
def comm(request):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2602_10056_b200 as wc

    c = wc.NshardComm.create(world=1, rank=0, transport=request.param)
    yield c
    c.close()


@pytest.mark.parametrize("block", [1, 16])
@pytest.mark.parametrize("n,r,dtype", [(5000, 40, "bf16"), (3001, 24, "f32"), (20000, 100, "bf16")])
def test_nshard_world1_matches_oracle(comm, n, r, dtype, block):
    import oracle
    import paper_2602_10056_b200 as wc
    from paper_2602_10056_b200.inputs import make_qkv

    Q, K, V = make_qkv(1, 2, 1, 300, n, 64, dtype, "G", seed=11)
    dev = torch.device("cuda:0")
    S = torch.empty(r, dtype=torch.int32, device=dev)
    R = torch.empty(1, dtype=torch.int32, device=dev)
    O = wc.forward_nshard(comm, Q.to(dev), K.to(dev), V.to(dev), r, n, 0, seed=3, S=S, r_eff=R, block=block)
    torch.cuda.synchronize()
    res = oracle.forward(Q.double().numpy(), K.double().numpy(), V.double().numpy(), r, seed=3, block=block)
    assert np.array_equal(S.cpu().numpy(), res["S"][0]) and int(R.cpu()[0]) == res["r_eff"][0]
    err = np.abs(O.float().cpu().numpy() - res["O"]).max() / np.abs(V.double().numpy()).max()
    assert err <= (2e-2 if dtype == "bf16" else 1e-4), err


def test_nshard_query_shard_and_rq(comm):
    # a query shard with R_Q supplied (Alg 2's explicit radius input)
    import oracle
    import paper_2602_10056_b200 as wc
    from paper_2602_10056_b200.inputs import make_qkv

    Q, K, V = make_qkv(1, 1, 1, 500, 4000, 128, "bf16", "C", seed=2)
    rq = float(torch.linalg.norm(Q.double(), dim=-1).max())
    dev = torch.device("cuda:0")
    Qs = Q[:, :, 100:350]
    S = torch.empty(64, dtype=torch.int32, device=dev)
    O = wc.forward_nshard(comm, Qs.to(dev), K.to(dev), V.to(dev), 64, 4000, 0, seed=5, rq=rq, S=S)
    torch.cuda.synchronize()
    res = oracle.forward(Q.double().numpy(), K.double().numpy(), V.double().numpy(), 64, seed=5, rq=rq)
    assert np.array_equal(S.cpu().numpy(), res["S"][0])
    err = np.abs(O.float().cpu().numpy()[0, 0] - res["O"][0, 0, 100:350]).max() / np.abs(V.double().numpy()).max()
    assert err <= 2e-2, err


@pytest.mark.parametrize("block", [1, 16])
def test_p2p_two_ranks_one_gpu(tmp_path, block):
    """The device-initiated transport across two processes (both on the one GPU of the test box:
    CUDA-IPC-mapped mailboxes, peer stores, system-scope flag release / acquire): the two-shard run
    selects the oracle's pivots and matches its outputs.  Shards are whole 2048-key chunks."""
    import socket
    import subprocess
    import sys

    import oracle
    from paper_2602_10056_b200.inputs import make_qkv

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "p2p.npz")
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, WC_T_BLOCK=str(block))
    procs = [subprocess.Popen([sys.executable, os.path.join(here, "nshard_p2p_worker.py"), str(k), "2", str(port), out],
                              env=env)
             for k in range(2)]
    try:
        rcs = [p.wait(timeout=240) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert rcs == [0, 0], rcs
    res = np.load(out)
    Q, K, V = make_qkv(1, 2, 1, 256, 8192, 64, "bf16", "G", seed=3)
    orc = oracle.forward(Q.double().numpy(), K.double().numpy(), V.double().numpy(), 24, seed=7, block=block)
    assert np.array_equal(res["S"], orc["S"][0]) and int(res["r_eff"][0]) == orc["r_eff"][0]
    err = np.abs(res["O"] - orc["O"]).max() / np.abs(V.double().numpy()).max()
    assert err <= 2e-2, err
