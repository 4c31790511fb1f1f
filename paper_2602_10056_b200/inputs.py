"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method: it only draws Q, K, V with the
shapes and value distributions of the paper's workloads (recipe in DESIGN.md
"Input recipe") and rounds them once to the config dtype.  The identical bytes
go to the GPU and (as exact float64 copies) to the oracle.

Families:
  G  i.i.d. N(0,1) queries, keys, values.
  C  clustered tokens (ViT / diffusion-like): 64 centres N(0,I); rows = centre + 0.3 N(0,I).
  L  LLM-like keys: N(0,I) + a per-channel offset 3 N(0,1) shared by the head's keys,
     4 outlier channels scaled x8 in K and x4 in Q.
  D  exactness family: keys drawn from `distinct` distinct N(0,I) vectors.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

DTYPES = {"f32": torch.float32, "bf16": torch.bfloat16}


@dataclass
class Config:
    name: str
    batch: int
    hq: int
    hkv: int
    m: int
    n: int
    d: int
    r: int
    dtype: str  # "f32" | "bf16"
    family: str = "G"
    seed: int = 0

    @property
    def units(self) -> int:
        return self.batch * self.hkv


# BASELINE.json configs (configs[0..4]) and the north-star headline.
CONFIGS = {
    "cfg1": Config("cfg1", 1, 1, 1, 256, 256, 16, 16, "f32"),
    "vit": Config("vit", 64, 12, 12, 197, 197, 64, 32, "bf16", "C"),
    "diffusion": Config("diffusion", 8, 16, 16, 4096, 4096, 64, 128, "bf16", "C"),
    "llm32k": Config("llm32k", 1, 32, 8, 32768, 32768, 128, 256, "bf16", "L"),
    "headline": Config("headline", 1, 1, 1, 65536, 65536, 128, 256, "bf16", "G"),
    # long-sequence sweep (configs[4]): one head, keys sharded along n over the GPUs
    "long256k": Config("long256k", 1, 1, 1, 262144, 262144, 128, 256, "bf16", "G"),
    "long1m": Config("long1m", 1, 1, 1, 1048576, 1048576, 128, 256, "bf16", "G"),
    "long4m": Config("long4m", 1, 1, 1, 4194304, 4194304, 128, 256, "bf16", "G"),
}

BLOCK_ROWS = 65536


def make_rows(n_rows_total: int, row0: int, count: int, d: int, dtype="bf16", seed=0, stream=0):
    """Rows [row0, row0 + count) of a long N(0,1) matrix generated in fixed 64K-row blocks, each from
    its own PCG64 stream: any shard of the sequence is reproducible without generating the rest."""
    out = np.empty((count, d))
    b0, b1 = row0 // BLOCK_ROWS, (row0 + count - 1) // BLOCK_ROWS
    for b in range(b0, b1 + 1):
        rng = np.random.Generator(np.random.PCG64([seed, stream, b]))
        blk = rng.standard_normal((min(BLOCK_ROWS, n_rows_total - b * BLOCK_ROWS), d))
        lo = max(row0, b * BLOCK_ROWS)
        hi = min(row0 + count, b * BLOCK_ROWS + blk.shape[0])
        out[lo - row0:hi - row0] = blk[lo - b * BLOCK_ROWS:hi - b * BLOCK_ROWS]
    return torch.from_numpy(out).to(DTYPES[dtype]).reshape(1, 1, count, d).contiguous()


def make_long_shard(cfg: Config, world: int, rank: int, seed=None):
    """(Q_shard, K_shard, V_shard, k_offset) of family-G inputs for the n-sharded path: keys/values
    [off, off + n_local) and an even query shard; identical global data for any world size."""
    seed = cfg.seed if seed is None else seed
    base, extra = divmod(cfg.n, world)
    off = rank * base + min(rank, extra)
    nl = base + (1 if rank < extra else 0)
    qb, qe = divmod(cfg.m, world)
    qoff = rank * qb + min(rank, qe)
    ml = qb + (1 if rank < qe else 0)
    Q = make_rows(cfg.m, qoff, ml, cfg.d, cfg.dtype, seed, 0)
    K = make_rows(cfg.n, off, nl, cfg.d, cfg.dtype, seed, 1)
    V = make_rows(cfg.n, off, nl, cfg.d, cfg.dtype, seed, 2)
    return Q, K, V, off


def _draw(rng: np.random.Generator, family: str, shape_q, shape_kv, d: int, distinct: int | None):
    b, hq, m, _ = shape_q
    _, hkv, n, _ = shape_kv
    if family == "G":
        Q = rng.standard_normal(shape_q)
        K = rng.standard_normal(shape_kv)
        V = rng.standard_normal(shape_kv)
    elif family == "C":
        cent = rng.standard_normal((64, d))
        Q = cent[rng.integers(0, 64, size=(b, hq, m))] + 0.3 * rng.standard_normal(shape_q)
        K = cent[rng.integers(0, 64, size=(b, hkv, n))] + 0.3 * rng.standard_normal(shape_kv)
        V = rng.standard_normal(shape_kv)
    elif family == "L":
        off = 3.0 * rng.standard_normal((b, hkv, 1, d))
        K = rng.standard_normal(shape_kv) + off
        Q = rng.standard_normal(shape_q)
        ch = rng.choice(d, size=min(4, d), replace=False)
        K[..., ch] *= 8.0
        Q[..., ch] *= 4.0
        V = rng.standard_normal(shape_kv)
    elif family == "D":
        k = distinct or 8
        base = rng.standard_normal((b, hkv, k, d))
        idx = rng.integers(0, k, size=(b, hkv, n))
        K = np.take_along_axis(base, idx[..., None].repeat(d, axis=-1), axis=2)
        Q = rng.standard_normal(shape_q)
        V = rng.standard_normal(shape_kv)
    else:
        raise ValueError(f"unknown family {family!r}")
    return Q, K, V


def make_qkv(batch, hq, hkv, m, n, d, dtype="bf16", family="G", seed=0, distinct=None):
    """Return (Q, K, V) as CPU torch tensors of `dtype` in the BHND layout
    ([batch, heads, seq, d]); float64 views of the same values via `.double()`."""
    rng = np.random.Generator(np.random.PCG64(seed))
    Q, K, V = _draw(rng, family, (batch, hq, m, d), (batch, hkv, n, d), d, distinct)
    tdt = DTYPES[dtype]
    return tuple(torch.from_numpy(np.ascontiguousarray(x)).to(tdt).contiguous() for x in (Q, K, V))


def make_config(cfg: Config, *, m=None, n=None, seed=None, family=None):
    return make_qkv(cfg.batch, cfg.hq, cfg.hkv, cfg.m if m is None else m, cfg.n if n is None else n,
                    cfg.d, cfg.dtype, cfg.family if family is None else family,
                    cfg.seed if seed is None else seed)


def query_sample(m: int, count: int, seed: int = 1234) -> np.ndarray:
    """Seeded sorted sample of query row indices (for full-size parity checks)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.sort(rng.choice(m, size=min(count, m), replace=False))
