"""fp64 CPU oracle for WildCat (arxiv 2602.10056) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2602_10056_b200``) never imports it and shares no code with it.

This module is argument marshalling (numpy -> ctypes) around ``wildcat_oracle.c``;
every arithmetic step lives in that C file, each function citing the PAPER.md
passage it follows.  Two helpers here are plain-definition *checkers* used by
the oracle's own pin tests (dense Nystrom residual, Lemma 2.1 right-hand side);
they are written from the paper's definitions with numpy and are not used by
the oracle itself.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wildcat_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_c_i32 = ctypes.c_int32
_c_i64 = ctypes.c_int64
_c_u64 = ctypes.c_uint64
_c_dbl = ctypes.c_double
_p = ctypes.c_void_p

# options of the prologue (the oracle's own constants, same meaning as the ABI's flags)
TAU_ONE = 2
NO_RECENTER = 4


def _flags(tau_one=False, recenter=True):
    return (TAU_ONE if tau_one else 0) | (0 if recenter else NO_RECENTER)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no FMA contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math",
            "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm",
        ])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            L.wco_philox4x32_10.argtypes = [_p, _p, _p]
            L.wco_pivot_uniform.argtypes = [_c_u64, ctypes.c_uint32, _c_u64]
            L.wco_pivot_uniform.restype = _c_dbl
            L.wco_lambert_w0.argtypes = [_c_dbl]
            L.wco_lambert_w0.restype = _c_dbl
            L.wco_rho0.restype = _c_dbl
            L.wco_temperature.argtypes = [_c_dbl, _c_dbl, _c_dbl, _c_i64]
            L.wco_temperature.restype = _c_dbl
            L.wco_prologue.argtypes = [_c_i64, _c_i32, _p, _c_i64, _p, _c_dbl, _c_dbl, _p, _p, _c_i32]
            L.wco_select.argtypes = [_c_i64, _c_i32, _c_i32, _p, _p, _c_dbl, _c_dbl, _c_u64, _c_u64,
                                     _p, _p, _p, _p, _p, _p]
            L.wco_select_mr.argtypes = [_c_i64, _c_i32, _c_i32, _p, _p, _c_dbl, _c_dbl, _c_u64, _c_u64,
                                        _p, _p, _p, _p, _p, _p]
            L.wco_weights.argtypes = [_c_i64, _c_i32, _c_i32, _p, _p, _p, _c_i32, _p, _c_dbl, _c_dbl, _p]
            L.wco_attend.argtypes = [_c_i64, _c_i32, _c_i32, _p, _p, _p, _c_i32, _c_dbl, _p, _p, _c_i32, _p]
            L.wco_exact_attention.argtypes = [_c_i64, _c_i64, _c_i32, _p, _p, _p, _c_dbl, _p]
            L.wco_forward.argtypes = [_c_i32, _c_i32, _c_i32, _c_i64, _c_i64, _c_i32, _c_i32, _c_dbl,
                                      _c_dbl, _c_u64, _c_i32, _c_i32, _p, _p, _p, _p, _p, _p, _p, _p, _c_u64, _c_i32]
            L.wco_forward_binned.argtypes = [_c_i32, _c_i32, _c_i32, _c_i64, _c_i64, _c_i32, _c_i32, _c_i32,
                                             _c_dbl, _c_dbl, _c_u64, _c_i32, _c_i32, _p, _p, _p, _p, _p, _p,
                                             _p, _p, _c_u64, _c_i32]
            L.wco_compress_kv.argtypes = [_c_i32, _c_i32, _c_i32, _c_i64, _c_i64, _c_i32, _c_i32, _c_i32, _c_i32,
                                          _c_i32, _c_i32, _c_dbl, _c_dbl, _c_u64, _p, _p, _p, _p, _p, _p, _p, _p,
                                          _p, _c_u64, _c_i32]
            L.wco_accept_uniform.argtypes = [_c_u64, ctypes.c_uint32, _c_u64]
            L.wco_accept_uniform.restype = _c_dbl
            L.wco_select_blocked.argtypes = [_c_i64, _c_i32, _c_i32, _c_i32, _p, _p, _c_dbl, _c_dbl, _c_u64,
                                             _c_u64, _p, _p, _p, _p, _p, _p, _p]
            L.wco_num_threads.restype = ctypes.c_int
            L.wco_set_num_threads.argtypes = [ctypes.c_int]
            _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_p)


# --------------------------------------------------------------------------- scalars
def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32).copy()
    k = np.asarray(key, dtype=np.uint32).copy()
    out = np.zeros(4, dtype=np.uint32)
    lib().wco_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def pivot_uniform(seed: int, round_i: int, unit: int) -> float:
    return lib().wco_pivot_uniform(seed, round_i, unit)


def lambert_w0(z: float) -> float:
    return lib().wco_lambert_w0(float(z))


def rho0() -> float:
    return lib().wco_rho0()


def temperature(beta, rq, rk, n) -> float:
    return lib().wco_temperature(float(beta), float(rq), float(rk), int(n))


def set_threads(t: int) -> None:
    lib().wco_set_num_threads(int(t))


def num_threads() -> int:
    return lib().wco_num_threads()


# --------------------------------------------------------------------------- per unit
def prologue(K, Qrows=None, rq=-1.0, beta=None, tau_one=False, recenter=True):
    K = _f64(K)
    n, d = K.shape
    beta = 1.0 / np.sqrt(d) if beta is None else float(beta)
    Qr = _f64(Qrows) if Qrows is not None else np.zeros((0, d))
    kbar = np.zeros(d)
    st = np.zeros(5)
    lib().wco_prologue(n, d, _ptr(K), Qr.shape[0], _ptr(Qr), float(rq), beta, _ptr(kbar), _ptr(st),
                       _flags(tau_one, recenter))
    return kbar, dict(tau=st[0], g=st[1], mstar=st[2], rk=st[3], rq=st[4])


def select(K, kbar, g, mstar, r, seed, unit=0):
    """F-form RPNys.  Returns dict(S, r_eff, F, p, trace, L)."""
    K = _f64(K)
    n, d = K.shape
    kbar = _f64(kbar)
    S = np.full(r, -1, dtype=np.int32)
    reff = np.zeros(1, dtype=np.int32)
    F = np.zeros((r, n))
    p = np.zeros(n)
    tr = np.full(r + 1, np.nan)
    L = np.zeros((r, r))
    rc = lib().wco_select(n, d, r, _ptr(K), _ptr(kbar), float(g), float(mstar), int(seed), int(unit),
                          _ptr(S), _ptr(reff), _ptr(F), _ptr(p), _ptr(tr), _ptr(L))
    if rc:
        raise MemoryError("wco_select failed")
    re = int(reff[0])
    return dict(S=S, r_eff=re, F=F, p=p, trace=tr[: re + 1], L=L)


def accept_uniform(seed, cand, unit=0):
    """Acceptance uniform of blocked-RPC candidate `cand` (Philox tag 'ACPT', reading Z22)."""
    return lib().wco_accept_uniform(int(seed), int(cand), int(unit))


def select_blocked(K, kbar, g, mstar, r, block, seed, unit=0):
    """Blocked (accelerated) RPCholesky, block size `block`.  Returns dict(S, r_eff, F, p, L, nblocks, ncand)."""
    K = _f64(K)
    n, d = K.shape
    kbar = _f64(kbar)
    S = np.full(r, -1, dtype=np.int32)
    reff = np.zeros(1, dtype=np.int32)
    F = np.zeros((r, n))
    p = np.zeros(n)
    L = np.zeros((r, r))
    nb = np.zeros(1, dtype=np.int32)
    nc = np.zeros(1, dtype=np.int32)
    rc = lib().wco_select_blocked(n, d, r, int(block), _ptr(K), _ptr(kbar), float(g), float(mstar), int(seed),
                                  int(unit), _ptr(S), _ptr(reff), _ptr(F), _ptr(p), _ptr(L), _ptr(nb), _ptr(nc))
    if rc:
        raise MemoryError("wco_select_blocked failed")
    return dict(S=S, r_eff=int(reff[0]), F=F, p=p, L=L, nblocks=int(nb[0]), ncand=int(nc[0]))


def select_mr(K, kbar, g, mstar, r, seed, unit=0):
    """Literal Alg 1 (M/R form).  Returns dict(S, r_eff, M, R, W, p)."""
    K = _f64(K)
    n, d = K.shape
    kbar = _f64(kbar)
    S = np.full(r, -1, dtype=np.int32)
    reff = np.zeros(1, dtype=np.int32)
    M = np.zeros((r, r))
    R = np.zeros((r, n))
    W = np.zeros((r, n))
    p = np.zeros(n)
    rc = lib().wco_select_mr(n, d, r, _ptr(K), _ptr(kbar), float(g), float(mstar), int(seed), int(unit),
                             _ptr(S), _ptr(reff), _ptr(M), _ptr(R), _ptr(W), _ptr(p))
    if rc:
        raise MemoryError("wco_select_mr failed")
    return dict(S=S, r_eff=int(reff[0]), M=M, R=R, W=W, p=p)


def weights(K, V, S, r_eff, kbar, g, mstar, r=None):
    K = _f64(K)
    V = _f64(V)
    n, d = K.shape
    S = np.ascontiguousarray(S, dtype=np.int32)
    r = len(S) if r is None else r
    X = np.zeros((r, d + 1))
    rc = lib().wco_weights(n, d, r, _ptr(K), _ptr(V), _ptr(S), int(r_eff), _ptr(_f64(kbar)),
                           float(g), float(mstar), _ptr(X))
    if rc == -2:
        raise np.linalg.LinAlgError("oracle Cholesky of H~_SS failed")
    if rc:
        raise MemoryError("wco_weights failed")
    return X


def attend(Q, KS, X, r_eff, beta, vmin, vmax, clip=True):
    Q = _f64(Q)
    m, d = Q.shape
    KS = _f64(KS)
    X = _f64(X)
    r = KS.shape[0]
    O = np.zeros((m, d))
    lib().wco_attend(m, d, r, _ptr(Q), _ptr(KS), _ptr(X), int(r_eff), float(beta),
                     _ptr(_f64(vmin)), _ptr(_f64(vmax)), int(bool(clip)), _ptr(O))
    return O


def exact_attention(Q, K, V, beta=None):
    Q = _f64(Q)
    K = _f64(K)
    V = _f64(V)
    m, d = Q.shape
    n = K.shape[0]
    beta = 1.0 / np.sqrt(d) if beta is None else float(beta)
    O = np.zeros((m, d))
    lib().wco_exact_attention(m, n, d, _ptr(Q), _ptr(K), _ptr(V), beta, _ptr(O))
    return O


def forward(Q, K, V, r, seed=0, beta=None, rq=-1.0, clip=True, block=1, bins=1, unit_offset=0, tau_one=False,
            recenter=True):
    """Alg 4 over [batch, heads, seq, d] arrays (float64 copies of the inputs).
    bins > 1: Alg 2 with B contiguous bins (wco_forward_binned; stats are then per bin).
    unit_offset: the units are [unit_offset, ...) of a larger batch (Philox unit ids, PAR2).

    Returns dict(O, S, r_eff, stats, X)."""
    if bins > 1:
        return forward_binned(Q, K, V, r, bins, seed=seed, beta=beta, rq=rq, clip=clip, block=block,
                              unit_offset=unit_offset, tau_one=tau_one, recenter=recenter)
    Q = _f64(Q)
    K = _f64(K)
    V = _f64(V)
    batch, hq, m, d = Q.shape
    _, hkv, n, _ = K.shape
    beta = 1.0 / np.sqrt(d) if beta is None else float(beta)
    units = batch * hkv
    O = np.zeros_like(Q)
    S = np.full((units, r), -1, dtype=np.int32)
    reff = np.zeros(units, dtype=np.int32)
    st = np.zeros((units, 5))
    X = np.zeros((units, r, d + 1))
    rc = lib().wco_forward(batch, hq, hkv, m, n, d, r, beta, float(rq), int(seed), int(bool(clip)), int(block),
                           _ptr(Q), _ptr(K), _ptr(V), _ptr(O), _ptr(S), _ptr(reff), _ptr(st), _ptr(X),
                           int(unit_offset), _flags(tau_one, recenter))
    if rc:
        raise RuntimeError(f"wco_forward failed ({rc})")
    return dict(O=O, S=S, r_eff=reff, stats=st, X=X)


def bin_rank(n, r, bins):
    """Per-bin rank rb = min(ceil(r / B), n / B) (reading Z13) and the coreset slots B * rb."""
    rb = min(-(-r // bins), n // bins)
    return rb, bins * rb


def forward_binned(Q, K, V, r, bins, seed=0, beta=None, rq=-1.0, clip=True, block=1, unit_offset=0, tau_one=False,
                   recenter=True):
    """Alg 4 with Alg 2 binning (wco_forward_binned).  Returns dict(O, S, r_eff, stats, X) with
    S [units][B*rb], stats [units][B][5] (tau_b, g_b, mstar_b, R_K^b, R_Q), X [units][B*rb][d+1]."""
    Q = _f64(Q)
    K = _f64(K)
    V = _f64(V)
    batch, hq, m, d = Q.shape
    _, hkv, n, _ = K.shape
    beta = 1.0 / np.sqrt(d) if beta is None else float(beta)
    units = batch * hkv
    _, R = bin_rank(n, r, bins)
    O = np.zeros_like(Q)
    S = np.full((units, R), -1, dtype=np.int32)
    reff = np.zeros(units, dtype=np.int32)
    st = np.zeros((units, bins, 5))
    X = np.zeros((units, R, d + 1))
    rc = lib().wco_forward_binned(batch, hq, hkv, m, n, d, r, bins, beta, float(rq), int(seed), int(bool(clip)),
                                  int(block), _ptr(Q), _ptr(K), _ptr(V), _ptr(O), _ptr(S), _ptr(reff), _ptr(st),
                                  _ptr(X), int(unit_offset), _flags(tau_one, recenter))
    if rc:
        raise RuntimeError(f"wco_forward_binned failed ({rc})")
    return dict(O=O, S=S, r_eff=reff, stats=st, X=X)


def kv_capacity(n, r, keep_first, keep_last, bins=1):
    """Cache rows per unit C = keep_first + keep_last + R (R = B*rb over the n_mid middle tokens)."""
    nmid = n - keep_first - keep_last
    R = bin_rank(nmid, r, bins)[1] if nmid > 0 else 0
    return keep_first + keep_last + R, R


def compress_kv(Q, K, V, r, keep_first=0, keep_last=0, bins=1, seed=0, beta=None, rq=-1.0, block=1, unit_offset=0,
                tau_one=False, recenter=True):
    """KV-cache compression (wco_compress_kv, reading Z24) over
    [batch, heads, seq, d] arrays.  Returns dict(KC [units][C][d], XC [units][C][d+1], c_eff [units],
    vmin, vmax [units][d], S [units][R] global token indices of the coreset)."""
    Q = _f64(Q)
    K = _f64(K)
    V = _f64(V)
    batch, hq, m, d = Q.shape
    _, hkv, n, _ = K.shape
    beta = 1.0 / np.sqrt(d) if beta is None else float(beta)
    units = batch * hkv
    C, R = kv_capacity(n, r, keep_first, keep_last, bins)
    KC = np.zeros((units, C, d))
    XC = np.zeros((units, C, d + 1))
    ceff = np.zeros(units, dtype=np.int32)
    vmin = np.zeros((units, d))
    vmax = np.zeros((units, d))
    S = np.full((units, max(R, 1)), -1, dtype=np.int32)
    rc = lib().wco_compress_kv(batch, hq, hkv, m, n, d, r, bins, int(block), int(keep_first), int(keep_last), beta,
                               float(rq), int(seed), _ptr(Q), _ptr(K), _ptr(V), _ptr(KC), _ptr(XC), _ptr(ceff),
                               _ptr(vmin), _ptr(vmax), _ptr(S), int(unit_offset), _flags(tau_one, recenter))
    if rc == -2:
        raise ValueError("invalid KV split (keep_first/keep_last/bins)")
    if rc:
        raise RuntimeError(f"wco_compress_kv failed ({rc})")
    return dict(KC=KC, XC=XC, c_eff=ceff, vmin=vmin, vmax=vmax, S=S[:, :R])


def cache_attend(Q, KC, XC, c_eff, vmin, vmax, hkv, beta=None, clip=True):
    """Alg 3 WtdAttn (wco_attend) of queries Q [batch, hq, m, d] over a compressed cache
    (KC, XC, c_eff, vmin, vmax per unit, units = batch*hkv); query head h uses unit h // (hq/hkv)."""
    Q = _f64(Q)
    batch, hq, m, d = Q.shape
    beta = 1.0 / np.sqrt(d) if beta is None else float(beta)
    group = hq // hkv
    O = np.zeros_like(Q)
    for b in range(batch):
        for h in range(hq):
            u = b * hkv + h // group
            O[b, h] = attend(Q[b, h], KC[u], XC[u], int(c_eff[u]), beta, vmin[u], vmax[u], clip=clip)
    return O


# --------------------------------------------------------------------------- checkers
def kernel_block(A, B, kbar, g, mstar):
    """h~(A, B) = exp(g <a-kbar, b-kbar> - mstar) as a dense block (numpy)."""
    A = _f64(A) - kbar
    B = _f64(B) - kbar
    return np.exp(g * (A @ B.T) - mstar)


def lemma21_rhs(A, Ahat, V):
    """Right-hand side of Lemma 2.1:
    ||V||_max * min( 3/sqrt(n) * ||A - Ahat||_{2->inf} / min_ij A_ij , 2 )."""
    n = A.shape[1]
    row = np.sqrt(((A - Ahat) ** 2).sum(axis=1)).max()
    return np.abs(V).max() * min(3.0 / np.sqrt(n) * row / A.min(), 2.0)
