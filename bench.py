#!/usr/bin/env python
"""bench.py -- WildCat coreset attention on B200: queries/s at n = 64K, d = 128, r = 256 (bf16).

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config headline] [--impl wildcat|reference]
One step = one pass of the whole hot path (prologue, RPCholesky selection, Nystrom weights,
weighted attend) over one batch of synthetic inputs resident in HBM, through the C ABI
(wildcat_forward).  L2 is flushed (a 512 MB write) before every timed step, outside the timed
events.  Multi-GPU (torchrun, PAR2): the config's (batch, kv-head) units are partitioned over the
ranks with no data-path collective, each rank passing unit_offset = its first unit so the pivots
are those of the one-GPU run (strong scaling); the 1-unit headline grows its batch with the ranks
instead (weak scaling).  Time = max over ranks.  --impl reference times the fp64 oracle.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "coreset-attention queries/s at n=64K,d=128,r=256; HBM GB/s; rel err vs exact"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# fp64 tensor-core (DMMA m8n8k4) throughput measured on this pool's B200 by tools/micro/fp64_bench.cu
# (profiles/r1_fp64_microbench.txt): there is no fp64 entry in MEASURED_PEAKS.json.
FP64_TENSOR_TFLOPS = 36.5


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def select_bytes(n, d, r, e, nblocks=None, fread=None):
    """Algorithmic HBM bytes of the selection loop per unit:
    per block (sequential: per round) the K rows (n d e) and the residual read + write (16 n), once
    the new F rows (8 n r), and the F prefix re-read at every block start (8 n Fread, Fread = sum of
    the block-start pivot counts).  Sequential RPC (nblocks = r, Fread = r (r-1) / 2) gives
    n r (d e + 24) + 4 n r (r - 1)."""
    if nblocks is None:
        nblocks, fread = r, r * (r - 1) / 2
    return n * (nblocks * (d * e + 16) + 8 * r + 8 * fread)


def cpu_oracle_sample(cfg, Q, K, V, block=1, bins=1, max_units=1):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload: the first `max_units`
    units run COMPLETELY (prologue, selection, weights, and the attend of every query row of the
    unit's q-heads) -- nothing is extrapolated: the rate is the queries actually answered divided by
    the seconds they took.  At the headline (1 unit) the sample is the whole workload.
    Returns (queries/s, seconds, details)."""
    import oracle

    threads = len(os.sched_getaffinity(0))
    oracle.set_threads(threads)
    group = cfg.hq // cfg.hkv
    nu = min(max_units, cfg.units)
    secs, queries = 0.0, 0
    for u in range(nu):
        b, h = divmod(u, cfg.hkv)
        Qu = Q[b:b + 1, h * group:(h + 1) * group].double().numpy()
        Ku = K[b:b + 1, h:h + 1].double().numpy()
        Vu = V[b:b + 1, h:h + 1].double().numpy()
        t0 = time.perf_counter()
        oracle.forward(Qu, Ku, Vu, cfg.r, seed=cfg.seed, block=block, bins=bins, unit_offset=u)
        secs += time.perf_counter() - t0
        queries += group * cfg.m
    what = f"Alg 4 (selection {'blocked b=' + str(block) if block >= 2 else 'sequential'}, B={bins})"
    info = dict(threads=threads, units=nu, queries=queries,
                sample=(f"oracle {what} on {nu} of {cfg.units} units, complete: prologue, selection, weights "
                        f"and the attend of all {group * cfg.m} query rows per unit; rate = queries answered / "
                        f"seconds (no extrapolation)"))
    return queries / secs, secs, info


def config_dict(cfg, args, world, mode, units_per_rank):
    """The `config` object of the JSON line -- identical for the GPU arm and the reference arm."""
    return {"workload": cfg.name, "units": cfg.units, "units_per_gpu": units_per_rank, "n": cfg.n, "m": cfg.m,
            "d": cfg.d, "r": cfg.r, "input_dtype": cfg.dtype, "family": cfg.family,
            "parallelism": (f"units{world}" if mode == "units" else f"nshard{world}-{args.transport}"),
            "select": "blocked" if args.block >= 2 else "sequential",
            "block": args.block, "bins": args.bins if mode == "units" else 1,
            "l2": f"flushed ({args.flush_mb} MB write) before each step"}


def unit_partition(cfg, world, rank):
    """PAR2 (P:303 ForPar; north_star "partitioned ... by (batch, head)"): the config's
    units split into contiguous ranges, one per rank, each run with unit_offset = its first unit (so
    every unit draws the Philox stream of the one-GPU run) -> strong scaling.  A config with fewer
    units than ranks (the 1-unit headline) instead grows the batch with the ranks: rank k holds unit
    k of a `world`-unit batch (inputs drawn with seed + k) -> weak scaling.
    Returns (u0, u1, unit_offset, scaling)."""
    U = cfg.units
    if U >= world and U % world == 0:
        per = U // world
        return rank * per, (rank + 1) * per, rank * per, "strong"
    return 0, U, rank * U, "weak"


def exact_errors(cfg, Qd, Kd, Vd, O):
    """max |O^ - O| / max |V| against fp64 exact attention (torch on the GPU, outside the timed region)
    on seeded query rows of up to 32 heads (P:144 normalisation)."""
    import torch

    from paper_2602_10056_b200.inputs import query_sample

    errs = []
    beta = 1.0 / math.sqrt(cfg.d)
    dev = Qd.device
    for b in range(cfg.batch):
        for h in range(cfg.hq):
            rows = torch.from_numpy(query_sample(cfg.m, 4096 // max(1, cfg.batch * cfg.hq) + 1, seed=b * 131 + h))
            q = Qd[b, h, rows.to(dev)].double()
            kk = Kd[b, h // (cfg.hq // cfg.hkv)].double()
            vv = Vd[b, h // (cfg.hq // cfg.hkv)].double()
            ex = torch.softmax(beta * (q @ kk.T), dim=-1) @ vv
            errs.append(float((O[b, h, rows.to(dev)].double() - ex).abs().max() / vv.abs().max()))
            if b * cfg.hq + h >= 31:
                break
        if len(errs) >= 32:
            break
    return errs


def kv_bins(target_rows, rb=12):
    """Bins B for the E3 setting B = r/12: r = target_rows coreset rows in bins of rb = 12
    (bins need not divide n_mid: the last bin takes the remainder, reading Z13)."""
    return max(1, target_rows // rb)


def kv_variant(dev, flush, block, steps, with_exact=True):
    """KV-cache workload (E3 protocol P:667-669, reading Z24) at the llm32k
    shapes (GQA 32/8, n = 32768, d = 128, bf16, L family): prefill compression keeping the first and
    last 32 tokens and compressing the rest so that the cache holds 25 % of the context, with
    B = r/12 bins (rb = 12; the last bin takes the remainder of n_mid, reading Z13), then
    one decode step (m = 1 new query per q-head) over the compressed cache vs exact decode attention
    over the full cache.  L2 flushed before every timed call."""
    import torch
    import torch.nn.functional as Fnn

    import paper_2602_10056_b200 as wc
    from paper_2602_10056_b200.inputs import CONFIGS, make_config, make_qkv

    cfg = CONFIGS["llm32k"]
    kf = kl = 32
    nmid = cfg.n - kf - kl
    bins = kv_bins(cfg.n // 4 - kf - kl)
    r = 12 * bins
    Q, K, V = make_config(cfg)
    Qd, Kd, Vd = Q.to(dev), K.to(dev), V.to(dev)
    del Q
    Qdec = make_qkv(cfg.batch, cfg.hq, cfg.hkv, 1, 16, cfg.d, cfg.dtype, cfg.family, seed=777)[0].to(dev)
    stream = torch.cuda.current_stream()

    def timed(fn, k):
        # a GPU-side sleep queued ahead of e0 keeps the device busy while the host enqueues fn, so
        # e0 -> e1 is device time (host launch latency excluded; a decode loop would be graph-captured)
        out, ts = None, []
        for _ in range(k):
            flush.zero_()
            torch.cuda._sleep(200000)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return out, ts

    comp = lambda: wc.compress_kv(Qd, Kd, Vd, r, keep_first=kf, keep_last=kl, bins=bins, block=block)
    comp()
    torch.cuda.synchronize()
    cache, tc = timed(comp, max(3, min(steps, 5)))
    dec = lambda: wc.attend(Qdec, cache)
    dec()
    Od, td = timed(dec, 30)
    exact = lambda: Fnn.scaled_dot_product_attention(Qdec, Kd, Vd, enable_gqa=True)
    exact()
    Oe, te = timed(exact, 30)
    C = cache.KC.shape[1]
    units = cfg.units
    cache_bytes = cache.nbytes + 2 * units * cfg.d * 2  # KC, VC (bf16), WC (fp32), value range
    kv_bytes = units * cfg.n * 2 * cfg.d * 2
    dec_us = statistics.median(td) * 1e3
    res = {"workload": "llm32k", "keep_first": kf, "keep_last": kl, "r": r, "bins": bins, "r_per_bin": 12,
           "block": block, "cache_rows_per_head": C, "c_eff_min": int(cache.r_eff.min().item()),
           "cache_bytes": cache_bytes, "kv_bytes": kv_bytes, "cache_fraction_of_kv_bytes": cache_bytes / kv_bytes,
           "compress_ms": statistics.median(tc), "decode_us": dec_us,
           "decode_steps_per_s": 1e6 / dec_us,
           "decode_cache_gbs": cache_bytes / (dec_us / 1e6) / 1e9,
           "exact_decode_sdpa_us": statistics.median(te) * 1e3,
           "timing": "CUDA events per call (device time: a queued GPU sleep hides host launch latency), L2 flushed before each; decode = one wildcat_attend (m = 1 per q-head, "
                     "all 32 q-heads) over the compressed cache; exact = torch SDPA over the full K, V"}
    if with_exact:
        beta = 1.0 / math.sqrt(cfg.d)
        errs = []
        g = cfg.hq // cfg.hkv
        for h in range(cfg.hq):
            q = Qdec[0, h].double()
            kk, vv = Kd[0, h // g].double(), Vd[0, h // g].double()
            ex = torch.softmax(beta * (q @ kk.T), dim=-1) @ vv
            errs.append(float((Od[0, h].double() - ex).abs().max() / vv.abs().max()))
        res["max_rel_err_vs_exact"] = max(errs)
        res["exact_sdpa_bf16_rel_err"] = max(
            float((Oe[0, h].double() - torch.softmax(1.0 / math.sqrt(cfg.d) * (Qdec[0, h].double()
                  @ Kd[0, h // g].double().T), -1) @ Vd[0, h // g].double()).abs().max() / Vd[0, h // g].double().abs().max())
            for h in range(cfg.hq))
    del cache, Qd, Kd, Vd
    torch.cuda.empty_cache()
    return res


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, cfg):
    """The reference arm: the fp64 oracle as it stands (the tier's reference), timed on the host cores,
    on the same workload/config as the GPU arm; each step a complete oracle run of a bounded sample
    (see cpu_oracle_sample).  Under torchrun only rank 0 runs; the others exit without work."""
    rank = _env_int("RANK", 0)
    if rank != 0:
        return
    from paper_2602_10056_b200.inputs import make_config

    world = max(1, args.gpus)
    mode = args.mode or ("nshard" if cfg.name.startswith("long") else "units")
    Q, K, V = make_config(cfg)
    block = args.block if mode == "units" else min(args.block, 16)
    for _ in range(args.warmup):
        cpu_oracle_sample(cfg, Q, K, V, block, args.bins)
    secs, queries = 0.0, 0
    info = None
    for _ in range(args.steps):
        _, s_, info = cpu_oracle_sample(cfg, Q, K, V, block, args.bins)
        secs += s_
        queries += info["queries"]
    value = queries / secs
    u0, u1, _, scaling = unit_partition(cfg, world, 0)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": scaling if mode == "units" else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, args, world, mode, u1 - u0),
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": info["threads"], "kind": "oracle",
                         "sample": info["sample"], "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="headline")
    ap.add_argument("--impl", default="wildcat", choices=["wildcat", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-exact", action="store_true", help="skip the accuracy-vs-exact and SDPA comparison")
    ap.add_argument("--flush-mb", type=int, default=512)
    ap.add_argument("--mode", default=None, choices=["units", "nshard"],
                    help="units: PAR2, the config's (batch, kv-head) units partitioned over the ranks (see "
                         "unit_partition); nshard: one sequence's keys sharded over the ranks (strong scaling). "
                         "Default: nshard for the long* configs, units otherwise")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"],
                    help="nshard mode: NCCL collectives, or device-initiated peer-memory mailboxes (8(f)-3)")
    ap.add_argument("--r", type=int, default=None, help="override the config's coreset size r")
    ap.add_argument("--n", type=int, default=None, help="override the config's n (= m)")
    ap.add_argument("--block", type=int, default=16,
                    help="pivot selection: 1 = sequential RPCholesky (Alg 1); b >= 2 = blocked RPCholesky "
                         "with b candidates per block (reading Z22; default 16)")
    ap.add_argument("--bins", type=int, default=1,
                    help="Alg 2 bins B (must divide n; default 1 = the north star's per-(batch, head) RPNys)")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip timing the other selection variant (sequential when --block >= 2)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)

    from paper_2602_10056_b200.inputs import CONFIGS, make_config

    cfg = CONFIGS[args.config]
    if args.r is not None or args.n is not None:
        import dataclasses

        cfg = dataclasses.replace(cfg, r=args.r or cfg.r, n=args.n or cfg.n, m=args.n or cfg.m,
                                  name=f"{cfg.name}_n{args.n or cfg.n}_r{args.r or cfg.r}")
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_2602_10056_b200 as wc
    from paper_2602_10056_b200 import _binding as B

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    mode = args.mode or ("nshard" if cfg.name.startswith("long") else "units")
    import dataclasses

    from paper_2602_10056_b200 import _binding as B0

    uoff, scaling, lcfg = 0, "strong", cfg
    if mode == "units":
        u0, u1, uoff, scaling = unit_partition(cfg, world, rank)
        per = u1 - u0
        if per == cfg.units:
            lcfg = cfg
        elif per % cfg.hkv == 0:  # whole batch elements
            lcfg = dataclasses.replace(cfg, batch=per // cfg.hkv)
        else:  # kv-heads (with their q-heads) of one batch element
            assert cfg.hkv % per == 0, "units per rank must tile batch elements or kv-head groups"
            g = cfg.hq // cfg.hkv
            lcfg = dataclasses.replace(cfg, batch=1, hkv=per, hq=per * g)
    units = lcfg.units

    rb_main, R_main = B0.coreset_rows(cfg.n, cfg.r, max(1, args.bins))
    S = torch.empty(units, max(cfg.r, R_main), dtype=torch.int32, device=dev)
    R = torch.empty(units, dtype=torch.int32, device=dev)
    flush = torch.empty(args.flush_mb * (1 << 20), dtype=torch.uint8, device=dev)
    if mode == "nshard":
        # one sequence, keys/values/queries sharded along the sequence over the ranks (strong scaling)
        from paper_2602_10056_b200.inputs import make_long_shard

        Q, K, V, koff = make_long_shard(cfg, world, rank)
        Qd, Kd, Vd = Q.to(dev), K.to(dev), V.to(dev)
        seed = cfg.seed
        comm = wc.NshardComm.create(transport=args.transport,
                                    capacity=max(cfg.r * (cfg.d + 1), 16 * (2 + cfg.d + cfg.r)) + 64)

        Obuf = torch.empty_like(Qd)

        def step():
            return wc.forward_nshard(comm, Qd, Kd, Vd, cfg.r, cfg.n, koff, seed=seed, S=S[0], r_eff=R, out=Obuf,
                                     block=min(args.block, 16))
    else:
        # PAR2: this rank's units of the batch (unit_partition), Philox ids from unit_offset = uoff
        seed = cfg.seed
        if scaling == "weak":  # the batch grows with the ranks: unit block `rank` drawn with seed + rank
            Q, K, V = make_config(cfg, seed=cfg.seed + rank)
        else:
            Qa, Ka, Va = make_config(cfg)
            if lcfg is cfg:
                Q, K, V = Qa, Ka, Va
            elif lcfg.batch * cfg.hkv == u1 - u0:
                b0 = u0 // cfg.hkv
                Q, K, V = (x[b0:b0 + lcfg.batch].contiguous() for x in (Qa, Ka, Va))
            else:
                b0, h0 = divmod(u0, cfg.hkv)
                g = cfg.hq // cfg.hkv
                Q = Qa[b0:b0 + 1, h0 * g:(h0 + lcfg.hkv) * g].contiguous()
                K, V = (x[b0:b0 + 1, h0:h0 + lcfg.hkv].contiguous() for x in (Ka, Va))
            del Qa, Ka, Va
        Qd, Kd, Vd = Q.to(dev), K.to(dev), V.to(dev)

        Obuf = torch.empty_like(Qd)  # preallocated: no allocator traffic inside the timed region

        def step():
            return wc.forward(Qd, Kd, Vd, cfg.r, seed=seed, S=S, r_eff=R, out=Obuf, block=args.block, bins=args.bins,
                              unit_offset=uoff)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = B.last_launch_count()

    B.timing_enable(True)
    stages = []
    step_ms = []
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    stream = torch.cuda.current_stream()
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        O = step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        stages.append(B.timing_read())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    B.timing_enable(False)

    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    queries_per_rank = lcfg.batch * lcfg.hq * cfg.m if mode == "units" else cfg.batch * cfg.hq * cfg.m / world
    value = queries_per_rank * world * args.steps / (total_ms / 1e3)

    # stage breakdown (ms, mean over timed steps): prologue, select, weights, attend
    st_names = ["prologue", "select", "weights", "attend"]
    st_mean = ([statistics.mean(s[i] for s in stages) for i in range(4)] if all(len(s) >= 4 for s in stages)
               else None)
    e = 2 if cfg.dtype == "bf16" else 4
    r_eff = int(R.min().item())
    sel_info = None
    if mode == "units":
        # selection bookkeeping of the same (deterministic) selection: blocks run, F rows re-read
        sel = wc.select(Qd, Kd, cfg.r, seed=seed, block=args.block, bins=args.bins, unit_offset=uoff)
        stt = sel.stats.double().cpu()  # per (unit, bin) sub-unit
        nb = cfg.n // args.bins
        Sh = sel.S.cpu().numpy()
        reff_b = [int(((Sh[su // args.bins] >= 0) & (Sh[su // args.bins] // nb == su % args.bins)).sum())
                  for su in range(units * args.bins)]
        alg_bytes = sum(select_bytes(nb, cfg.d, reff_b[su], e, float(stt[su, 6]), float(stt[su, 8]))
                        for su in range(units * args.bins))
        # algorithmic fp64 flops of the round updates: kernel dots 2 n d r_eff + F-prefix dots 2 n Fdot
        alg_flops = sum(2.0 * nb * (cfg.d * reff_b[su] + float(stt[su, 9])) for su in range(units * args.bins))
        sel_info = {"block": args.block, "bins": args.bins, "blocks_per_unit": float(stt[:, 6].mean()),
                    "candidates_per_unit": float(stt[:, 7].mean()), "f_rows_reread_per_unit": float(stt[:, 8].mean()),
                    "alg_fp64_flops": alg_flops}
        del sel
    else:
        alg_bytes = units * select_bytes(cfg.n, cfg.d, r_eff, e)
    sel_ms = st_mean[1] if st_mean else None
    achieved = alg_bytes / (sel_ms / 1e3) / 1e9 if sel_ms else None
    peak, peak_kind = peaks()
    roof64 = None
    if sel_info and sel_ms:
        a64 = sel_info["alg_fp64_flops"] / (sel_ms / 1e3) / 1e12
        roof64 = {"kernel": "rpc_select_blocked_kernel" if args.block >= 2 else "rpc_select_tma_kernel",
                  "bound": "fp64", "achieved": a64, "peak": FP64_TENSOR_TFLOPS, "peak_kind":
                  "measured DMMA microbenchmark (tools/micro/fp64_bench.cu)", "unit": "TFLOP/s",
                  "frac": a64 / FP64_TENSOR_TFLOPS}

    # the other selection variant on the same inputs (context: sequential Alg 1 vs blocked)
    variants = None
    if not args.no_variants and mode == "units" and args.block >= 2:
        nvs = max(2, min(5, args.steps))
        forward_seq = lambda: wc.forward(Qd, Kd, Vd, cfg.r, seed=seed, S=S, r_eff=R, out=Obuf, block=1,
                                         unit_offset=uoff)
        forward_seq()
        torch.cuda.synchronize()
        B.timing_enable(True)
        vt, vst = [], []
        for _ in range(nvs):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            forward_seq()
            e1.record(stream)
            e1.synchronize()
            vt.append(e0.elapsed_time(e1))
            vst.append(B.timing_read())
        B.timing_enable(False)
        vsel = statistics.mean(x[1] for x in vst)
        vbytes = units * select_bytes(cfg.n, cfg.d, int(R.min().item()), e)
        variants = {"sequential": {"block": 1, "bins": args.bins, "steps": nvs, "ms_per_step": statistics.mean(vt),
                                   "queries_per_s": queries_per_rank * world / (statistics.mean(vt) / 1e3),
                                   "select_ms": vsel, "select_hbm_gbs": vbytes / (vsel / 1e3) / 1e9,
                                   "select_hbm_frac": vbytes / (vsel / 1e3) / 1e9 / peak}}
    # Alg 2 binning with the paper's KV-cache setting B ~ r/12: the largest power of two
    # <= r/12 that divides n (so B = 16 at the headline), blocked selection, same inputs
    if not args.no_variants and mode == "units" and args.bins == 1:
        bv = 1
        while bv * 2 <= max(1, cfg.r // 12) and cfg.n % (bv * 2) == 0:
            bv *= 2
        if bv > 1:
            _, Rv = B0.coreset_rows(cfg.n, cfg.r, bv)
            Sv = torch.empty(units, Rv, dtype=torch.int32, device=dev)
            fwd_b = lambda: wc.forward(Qd, Kd, Vd, cfg.r, seed=seed, S=Sv, r_eff=R, out=Obuf, block=max(2, args.block),
                                       bins=bv, unit_offset=uoff)
            fwd_b()
            torch.cuda.synchronize()
            vt = []
            for _ in range(max(2, min(5, args.steps))):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fwd_b()
                e1.record(stream)
                e1.synchronize()
                vt.append(e0.elapsed_time(e1))
            Ob = fwd_b()
            torch.cuda.synchronize()
            berr = max(exact_errors(lcfg, Qd, Kd, Vd, Ob)) if (rank == 0 and not args.no_exact) else None
            variants = variants or {}
            variants["binned"] = {"bins": bv, "block": max(2, args.block), "r_per_bin": Rv // bv,
                                  "ms_per_step": statistics.mean(vt),
                                  "queries_per_s": queries_per_rank * world / (statistics.mean(vt) / 1e3),
                                  "max_rel_err_vs_exact": berr}
    # KV-cache workload (prefill compression + decode) at the LLM shapes, rank 0, single GPU
    if not args.no_variants and mode == "units" and rank == 0 and world == 1 and args.config == "headline":
        variants = variants or {}
        variants["kvcache"] = kv_variant(dev, flush, max(2, args.block), args.steps, with_exact=not args.no_exact)
    # A5 against its own roofline (HBM-bound for r < 258 at bf16; intensity ~ r flop/byte):
    # algorithmic bytes 2 m d e + r d e + 4 r (d + 1) per head and flops 4 m r d, over the attend stage
    attend_roof = None
    if st_mean and mode == "units":
        at_ms = st_mean[3]
        heads = lcfg.batch * lcfg.hq
        a_bytes = heads * 2 * cfg.m * cfg.d * e + units * (R_main * cfg.d * e + 4 * R_main * (cfg.d + 1))
        a_flops = heads * 4.0 * cfg.m * R_main * cfg.d
        tp = None
        ws_path = os.environ.get("WC_ATTEND") not in ("tc", "cuda") and cfg.dtype == "bf16" and cfg.d in (64, 128)
        tpf = os.path.join(ROOT, "profiles", "r2_ncu_attend_ws_headline_summary.txt" if ws_path
                           else "r1_ncu_attend_full_summary.txt")
        if cfg.name == "headline" and os.path.exists(tpf):
            for ln in open(tpf):
                if ln.startswith("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"):
                    tp = float(ln.split()[1]) / 100.0
        attend_roof = {"kernel": "attend_ws_kernel (+ attend_long_prep_kernel)" if ws_path
                       else "attend_tc_kernel (+ attend_img_prep_kernel)", "bound": "hbm",
                       "achieved": a_bytes / (at_ms / 1e3) / 1e9, "peak": peaks()[0], "unit": "GB/s",
                       "frac": a_bytes / (at_ms / 1e3) / 1e9 / peaks()[0],
                       "tflops": a_flops / (at_ms / 1e3) / 1e12, "tensor_peak_tflops": 1685.2,
                       "tensor_pipe_active_ncu": tp}
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"select_traffic_{cfg.name}" + (f"_b{args.block}" if args.block >= 2 else "")
                      + ".json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # end to end through the public API with host buffers (pinned), H2D + forward + D2H per step
    e2e = None
    if not args.no_e2e and mode == "units":
        Qh, Kh, Vh = (x.pin_memory() for x in (Q, K, V))
        for _ in range(max(1, args.warmup)):
            wc.forward_host(Qh, Kh, Vh, cfg.r, seed=seed, device=dev, block=args.block, unit_offset=uoff)
        tt = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            wc.forward_host(Qh, Kh, Vh, cfg.r, seed=seed, device=dev, block=args.block, unit_offset=uoff)
            tt.append(time.perf_counter() - t0)
        te = torch.tensor([sum(tt)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        h2d = sum(x.numel() * x.element_size() for x in (Q, K, V))
        d2h = O.numel() * O.element_size()
        serial = queries_per_rank * world * args.steps / float(te.item())
        # streamed: HostPipeline (public API) over the same host batches -- per step H2D of Q, K, V,
        # wildcat_forward, D2H of O, on three event-ordered streams over two device slots, so the copies
        # of neighbouring steps overlap the compute; wall clock from the first submit to the last result
        pipe = wc.HostPipeline(Qh, Kh, cfg.r, seed=seed, device=dev, block=args.block, unit_offset=uoff)
        outs = [torch.empty(O.shape, dtype=O.dtype, pin_memory=True) for _ in range(2)]
        for k in range(max(2, args.warmup)):
            pipe.submit(Qh, Kh, Vh, outs[k % 2])
        pipe.synchronize()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(args.steps):
            pipe.submit(Qh, Kh, Vh, outs[k % 2])
        pipe.synchronize()
        tp = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tp, op=dist.ReduceOp.MAX)
        e2e = {"value": queries_per_rank * world * args.steps / float(tp.item()), "unit": "queries/s",
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
               "timing": ("host wall clock from the first submit to the last result of a HostPipeline over pinned "
                          "host batches: per step H2D of Q, K, V, wildcat_forward, D2H of O, the copies of "
                          "neighbouring steps overlapping the compute (no L2 flush: every step's 50 MB of inputs "
                          "is re-copied from the host)"),
               "serial_value": serial,
               "serial_timing": ("host wall clock around each forward_host call (H2D of K, Q; wildcat_select with "
                                 "the H2D of V overlapped; wildcat_weights; wildcat_attend; D2H of O; sync), L2 "
                                 "flushed before each")}

    # accuracy vs exact attention (the metric's third part) on 4096 seeded query rows, fp64 on the
    # GPU (torch matmul; a measurement helper outside the timed region), and the exact bf16 SDPA
    # time on the same shape for context (B = 1 WildCat is slower than exact attention below
    # n ~ 262K at r = 256 -- SURVEY.md 8(d)).
    err = None
    sdpa_ms = None
    if rank == 0 and mode == "units" and not args.no_exact:
        from paper_2602_10056_b200.inputs import query_sample

        O_ref = step()
        torch.cuda.synchronize()
        errs = exact_errors(lcfg, Qd, Kd, Vd, O_ref)
        err = {"max_rel_err_vs_exact": max(errs), "rows_per_head": 4096 // max(1, lcfg.batch * lcfg.hq) + 1,
               "heads_checked": len(errs), "norm": "max|O^ - O| / max|V| (P:144)"}
        try:
            import torch.nn.functional as Fnn

            for _ in range(2):
                Fnn.scaled_dot_product_attention(Qd, Kd, Vd, enable_gqa=lcfg.hq != lcfg.hkv)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            tt = []
            for _ in range(3):
                flush.zero_()
                e0.record()
                Fnn.scaled_dot_product_attention(Qd, Kd, Vd, enable_gqa=lcfg.hq != lcfg.hkv)
                e1.record()
                e1.synchronize()
                tt.append(e0.elapsed_time(e1))
            sdpa_ms = statistics.median(tt)
        except Exception:
            sdpa_ms = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and cfg.n <= 262144:
        v, secs, info = cpu_oracle_sample(lcfg, Q, K, V, block=args.block, bins=args.bins)
        cpu = {"value": v, "unit": "queries/s", "cores": info["threads"], "kind": "oracle",
               "sample": info["sample"], "cpu": cpu_model(), "seconds": secs}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "queries/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps,
            "higher_is_better": True,
            "scaling": scaling if mode == "units" else "strong",
            "vs_baseline": None,
            "dtype": "f64-select/f32-gemm",
            "data": "synthetic",
            "config": config_dict(cfg, args, world, mode, units),
            "r_eff_min": r_eff,
            "unit_offset": uoff,
            "stages_ms": dict(zip(st_names, st_mean)) if st_mean else None,
            "selection": sel_info,
            "roofline_fp64": roof64,
            "variants": variants,
            "roofline": {"kernel": "rpc_select_blocked_kernel" if args.block >= 2 else "rpc_select_tma_kernel",
                         "bound": "hbm", "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak if achieved else None,
                         "traffic": traffic,
                         "alg_bytes_per_launch": alg_bytes},
            "roofline_attend": attend_roof,
            "accuracy": err,
            "exact_sdpa_bf16_ms": sdpa_ms,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if mode == "nshard":
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
