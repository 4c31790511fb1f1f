"""PAR2 host logic ("ForPar"; north_star "partitioned across the GPUs of one box
by (batch, head), which needs no collectives") on CPU with world-size-2 gloo process groups.

Each rank takes its contiguous unit range from bench.unit_partition, slices the config's inputs the
way bench.py does and runs the fp64 oracle on its slice with unit_offset = its first unit; the
gathered per-rank results must equal the one-process run over all units bit for bit (pivots, r_eff
and outputs).  The GPU side of the same property (unit_offset in the C ABI) is
tests/test_gpu_options.py::test_unit_offset_partition_bitwise."""
import dataclasses
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfgs():
    from paper_2602_10056_b200.inputs import Config

    return {
        # diffusion-like: units = batch x heads, partitioned by batch elements
        "batched": Config("batched", 4, 2, 2, 48, 160, 16, 12, "f32", "C"),
        # LLM-like GQA: one batch element, kv-heads (with their q-heads) partitioned
        "gqa": Config("gqa", 1, 8, 4, 40, 200, 16, 10, "f32", "L"),
    }


def _slice(cfg, u0, u1, Q, K, V):
    per = u1 - u0
    if per == cfg.units:
        return Q, K, V
    if per % cfg.hkv == 0:
        b0 = u0 // cfg.hkv
        nb = per // cfg.hkv
        return Q[b0:b0 + nb], K[b0:b0 + nb], V[b0:b0 + nb]
    b0, h0 = divmod(u0, cfg.hkv)
    g = cfg.hq // cfg.hkv
    return Q[b0:b0 + 1, h0 * g:(h0 + per) * g], K[b0:b0 + 1, h0:h0 + per], V[b0:b0 + 1, h0:h0 + per]


def _worker(rank, world, port, name, block, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import oracle
        from paper_2602_10056_b200.inputs import make_config

        cfg = _cfgs()[name]
        u0, u1, uoff, scaling = bench.unit_partition(cfg, world, rank)
        Q, K, V = (x.double().numpy() for x in make_config(cfg))
        Qs, Ks, Vs = _slice(cfg, u0, u1, Q, K, V)
        res = oracle.forward(Qs, Ks, Vs, cfg.r, seed=cfg.seed, block=block, unit_offset=uoff)
        # gather (S, r_eff, O) of every rank: no data-path collective in the method, this is the check
        S = [torch.zeros((u1 - u0, cfg.r), dtype=torch.int32) for _ in range(world)]
        dist.all_gather(S, torch.from_numpy(res["S"]))
        O = [torch.zeros(Qs.shape, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(O, torch.from_numpy(res["O"]))
        if rank == 0:
            full = oracle.forward(Q, K, V, cfg.r, seed=cfg.seed, block=block)
            Sg = np.concatenate([s.numpy() for s in S], 0)
            ok_s = np.array_equal(Sg, full["S"])
            Og = np.concatenate([o.numpy() for o in O], 0 if Qs.shape[0] != Q.shape[0] else 1)
            ok_o = np.array_equal(Og, full["O"])
            q.put((scaling, ok_s, ok_o))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["batched", "gqa"])
@pytest.mark.parametrize("block", [1, 4])
def test_par2_partition_world2(name, block):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, block, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    scaling, ok_s, ok_o = q.get(timeout=10)
    assert scaling == "strong"
    assert ok_s, "partitioned pivots differ from the one-process run"
    assert ok_o, "partitioned outputs differ from the one-process run"


def test_unit_partition_rules():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2602_10056_b200.inputs import CONFIGS

    # diffusion: 128 units over 1/2/4/8 GPUs -> contiguous equal ranges, offsets = first unit
    cfg = CONFIGS["diffusion"]
    for w in (1, 2, 4, 8):
        ranges = [bench.unit_partition(cfg, w, r) for r in range(w)]
        assert [a for a, _, _, _ in ranges] == [r * 128 // w for r in range(w)]
        assert all(off == a and sc == "strong" for a, _, off, sc in ranges)
        assert ranges[-1][1] == 128
    # LLM: 8 kv-heads over 8 GPUs -> one kv-head (4 q-heads) each
    cfg = CONFIGS["llm32k"]
    assert [bench.unit_partition(cfg, 8, r)[:3] for r in range(8)] == [(r, r + 1, r) for r in range(8)]
    # the 1-unit headline grows its batch: rank k holds unit k (weak scaling)
    cfg = CONFIGS["headline"]
    assert [bench.unit_partition(cfg, 4, r) for r in range(4)] == [(0, 1, r, "weak") for r in range(4)]
    lcfg = dataclasses.replace(cfg)
    assert lcfg.units == 1
