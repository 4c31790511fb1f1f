"""Host-side logic of the n-sharded path (PAR3) on CPU with world-size-2 gloo process groups.

The CUDA kernels cannot run here, so this test emulates the per-round protocol of nshard.cu in
numpy (fp64) on each rank -- shard ranges, prologue all-reduces (column sums, max norms, n_global
in Eq. 7), per-rank residual totals all-gathered, owner rank by prefix, owner-local inverse CDF,
pivot packet summed across ranks -- and checks that the sharded run selects exactly the pivots of
the unsharded fp64 oracle (Alg 1) for the same Philox stream."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CHUNK = 2048


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(x, op=dist.ReduceOp.SUM):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t, op=op)
    return t.numpy()


def _allgather_scalar(v, world):
    out = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(out, torch.tensor([v], dtype=torch.float64))
    return np.array([o.item() for o in out])


def _inverse_cdf(vals, t):
    acc = 0.0
    for idx, v in enumerate(vals):
        if acc + v > t:
            return idx, acc
        acc += v
    last = max(i for i, v in enumerate(vals) if v > 0)
    return last, sum(vals[:last])


def _rank_main(rank, world, port, n, d, r, seed, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2602_10056_b200 as wc
    from paper_2602_10056_b200.inputs import make_qkv

    Q, K, V = make_qkv(1, 1, 1, 64, n, d, "bf16", "G", seed=seed)
    Kg = K[0, 0].double().numpy()
    off, nl = wc.shard_range(n, world, rank)
    Kl = Kg[off:off + nl]
    Ql = Q[0, 0].double().numpy()[rank::world]  # a query shard
    beta = 1 / math.sqrt(d)
    # prologue reductions
    kbar = _allreduce(Kl.sum(0)) / n
    rq = math.sqrt(_allreduce(np.array([(Ql ** 2).sum(1).max()]), dist.ReduceOp.MAX)[0])
    kc = Kl - kbar
    rk = math.sqrt(_allreduce(np.array([(kc ** 2).sum(1).max()]), dist.ReduceOp.MAX)[0])
    tau = oracle.temperature(beta, rq, rk, n)
    g = beta / tau ** 2
    mstar = g * rk * rk
    p = np.exp(g * (kc ** 2).sum(1) - mstar)
    F = np.zeros((r, nl))
    S = []
    T0 = theta = None
    for i in range(r):
        chunks = [p[c:c + CHUNK].sum() for c in range(0, nl, CHUNK)]
        totals = _allgather_scalar(sum(chunks), world)
        T = totals.sum()
        if i == 0:
            T0, theta = T, 1000.0 * r * 2.0 ** -52 * T
        if T <= theta:
            break
        t = oracle.pivot_uniform(seed, i, 0) * T
        owner, excl = _inverse_cdf(list(totals), t)
        packet = np.zeros(2 + d + r)
        if owner == rank:
            c, cex = _inverse_cdf(chunks, t - excl)
            s_loc, sex = _inverse_cdf(list(p[c * CHUNK:(c + 1) * CHUNK]), t - excl - cex)
            s_loc += c * CHUNK
            packet[0], packet[1] = off + s_loc, p[s_loc]
            packet[2:2 + d] = Kl[s_loc]
            packet[2 + d:2 + d + i] = F[:i, s_loc]
        packet = _allreduce(packet)
        s_glob, ps = int(packet[0]), packet[1]
        kcs = packet[2:2 + d] - kbar
        fs = packet[2 + d:2 + d + i]
        col = np.exp(g * (kc @ kcs) - mstar) - F[:i].T @ fs
        F[i] = col / math.sqrt(ps)
        p = np.maximum(p - F[i] ** 2, 0.0)
        if off <= s_glob < off + nl:
            p[s_glob - off] = 0.0
        S.append(s_glob)
    ret[rank] = S
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_protocol_reproduces_oracle_pivots(world):
    n, d, r, seed = 5000, 16, 24, 7
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_rank_main, args=(world, port, n, d, r, seed, ret), nprocs=world, join=True)
    import oracle
    from paper_2602_10056_b200.inputs import make_qkv

    Q, K, V = make_qkv(1, 1, 1, 64, n, d, "bf16", "G", seed=seed)
    K64 = K[0, 0].double().numpy()
    kbar, st = oracle.prologue(K64, Q[0, 0].double().numpy())
    ref = oracle.select(K64, kbar, st["g"], st["mstar"], r, seed=seed, unit=0)
    for rk in range(world):
        assert ret[rk] == list(ref["S"][: ref["r_eff"]]), (rk, ret[rk], ref["S"])


def test_shard_range_partitions():
    import paper_2602_10056_b200 as wc

    for n in [1, 7, 2048, 100003]:
        for world in [1, 2, 3, 8]:
            if world > n:
                continue
            parts = [wc.shard_range(n, world, q) for q in range(world)]
            assert parts[0][0] == 0 and all(nl >= 1 for _, nl in parts)
            assert all(parts[q][0] + parts[q][1] == parts[q + 1][0] for q in range(world - 1))
            assert parts[-1][0] + parts[-1][1] == n


def _rank_main_blocked(rank, world, port, n, d, r, b, seed, ret):
    """The blocked n-sharded protocol of nshard.cu (ns_blk_pick / elim / update), in numpy: per block
    the rank totals are all-gathered, every rank draws the b candidates from the GLOBAL residual and
    the owners fill their packets {s, p_s, k_s, F[0:i, s]}, the packets are all-reduced, every rank
    runs the same rejection (reading Z22) on H = h~(K_C, K_C) - F_C^T F_C, then the accepted rounds
    update its own keys."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2602_10056_b200 as wc
    from paper_2602_10056_b200.inputs import make_qkv

    Q, K, V = make_qkv(1, 1, 1, 64, n, d, "bf16", "G", seed=seed)
    Kg = K[0, 0].double().numpy()
    off, nl = wc.shard_range(n, world, rank)
    Kl = Kg[off:off + nl]
    Ql = Q[0, 0].double().numpy()[rank::world]
    beta = 1 / math.sqrt(d)
    kbar = _allreduce(Kl.sum(0)) / n
    rq = math.sqrt(_allreduce(np.array([(Ql ** 2).sum(1).max()]), dist.ReduceOp.MAX)[0])
    kc = Kl - kbar
    rk = math.sqrt(_allreduce(np.array([(kc ** 2).sum(1).max()]), dist.ReduceOp.MAX)[0])
    tau = oracle.temperature(beta, rq, rk, n)
    g = beta / tau ** 2
    mstar = g * rk * rk
    p = np.exp(g * (kc ** 2).sum(1) - mstar)
    F = np.zeros((r, nl))
    S = []
    i, cbase, blk = 0, 0, 0
    theta = None
    plen = 2 + d + r
    while i < r:
        chunks = [p[c:c + CHUNK].sum() for c in range(0, nl, CHUNK)]
        totals = _allgather_scalar(sum(chunks), world)
        T = totals.sum()
        if blk == 0:
            theta = 1000.0 * r * 2.0 ** -52 * T
        if T <= theta:
            break
        packets = np.zeros(b * plen)
        for j in range(b):
            t = oracle.pivot_uniform(seed, cbase + j, 0) * T
            owner, excl = _inverse_cdf(list(totals), t)
            if owner == rank:
                c, cex = _inverse_cdf(chunks, t - excl)
                s_loc, _ = _inverse_cdf(list(p[c * CHUNK:(c + 1) * CHUNK]), t - excl - cex)
                s_loc += c * CHUNK
                pk = packets[j * plen:(j + 1) * plen]
                pk[0], pk[1] = off + s_loc, p[s_loc]
                pk[2:2 + d] = Kl[s_loc]
                pk[2 + d:2 + d + i] = F[:i, s_loc]
        packets = _allreduce(packets).reshape(b, plen)
        sg = packets[:, 0].astype(np.int64)
        kcs = packets[:, 2:2 + d] - kbar
        fc = packets[:, 2 + d:2 + d + i]
        H = np.exp(g * (kcs @ kcs.T) - mstar) - fc @ fc.T
        np.fill_diagonal(H, packets[:, 1])
        acc, rinv, Fc = [], [], []
        for j in range(b):
            if i + len(acc) >= r:
                break
            v = oracle.accept_uniform(seed, cbase + j, 0)
            if sg[j] not in [sg[a] for a in acc] and v * packets[j, 1] < H[j, j]:
                ri = 1.0 / math.sqrt(H[j, j])
                fj = H[j] * ri  # F[i + len(acc), s_e] for the later candidates e
                Fc.append(np.where(np.arange(b) > j, fj, 0.0))
                H = H - np.outer(fj, fj)
                acc.append(j)
                rinv.append(ri)
        na = len(acc)
        # the accepted rounds on the local keys (ns_blk_update): kernel column minus the F prefix
        # (read once for the block), then the per-key triangle with the elimination's coefficients
        G = np.stack([np.exp(g * (kc @ kcs[j]) - mstar) - F[:i].T @ fc[j] for j in acc]) if na else np.zeros((0, nl))
        for a, j in enumerate(acc):
            row = G[a].copy()
            for a2 in range(a):
                row -= F[i + a2] * Fc[a2][j]  # Fx[a][a2] = F[i + a2, s_a]
            F[i + a] = row * rinv[a]
            p = np.maximum(p - F[i + a] ** 2, 0.0)
            s_glob = int(sg[j])
            if off <= s_glob < off + nl:
                p[s_glob - off] = 0.0
            S.append(s_glob)
        i += na
        cbase += b
        blk += 1
    ret[rank] = S[:r]
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_blocked_sharded_protocol_reproduces_oracle_pivots(world):
    n, d, r, b, seed = 5000, 16, 24, 8, 7
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_rank_main_blocked, args=(world, port, n, d, r, b, seed, ret), nprocs=world, join=True)
    import oracle
    from paper_2602_10056_b200.inputs import make_qkv

    Q, K, V = make_qkv(1, 1, 1, 64, n, d, "bf16", "G", seed=seed)
    K64 = K[0, 0].double().numpy()
    kbar, st = oracle.prologue(K64, Q[0, 0].double().numpy())
    ref = oracle.select_blocked(K64, kbar, st["g"], st["mstar"], r, b, seed=seed, unit=0)
    for rk in range(world):
        assert ret[rk] == list(ref["S"][: ref["r_eff"]]), (rk, ret[rk], ref["S"])
