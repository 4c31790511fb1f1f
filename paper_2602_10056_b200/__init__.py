"""paper_2602_10056_b200 -- WildCat weighted-coreset attention on NVIDIA B200.

Public API (torch tensors in the BHND layout [batch, heads, seq, d], CUDA only):

    O = forward(Q, K, V, r, seed=0)                         # Alg 4 WildCat
    sel = select(Q, K, r, seed=0)                           # Alg 2 lines 1-6 + Alg 1 (RPNys)
    cache = weights(K, V, sel)                              # Alg 2 "Compress values"
    O = attend(Q, cache)                                    # Alg 3 WtdAttn
    O = forward_host(Q_cpu, K_cpu, V_cpu, r)                # host buffers in, host result out
    pipe = HostPipeline(Q_cpu, K_cpu, r); pipe.submit(Qh, Kh, Vh, Oh)  # streamed host batches, copies overlapped
    cache = compress_kv(Q, K, V, r, keep_first=32, keep_last=32)  # KV-cache compression (prefill)
    O_new = attend(Q_new, cache)                            # decode over the compressed cache
    comm = NshardComm.create(group)                         # keys of one sequence sharded over ranks
    O_loc = forward_nshard(comm, Q_loc, K_loc, V_loc, r, n_global, n_offset)

Everything runs in libwildcat.so (hand-written sm_100a kernels behind a C ABI,
include/wildcat.h).  There is no CPU fallback: CPU tensors raise (except
forward_host, which only copies host<->device around the same CUDA call).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _binding as B
from ._binding import NonFiniteInput, WildcatError, lib  # noqa: F401

__all__ = ["forward", "forward_host", "HostForward", "HostPipeline", "select", "weights", "attend", "decode", "Selection", "Cache",
           "KvCache", "WildcatError",
           "STATS_STRIDE", "NshardComm", "forward_nshard", "shard_range", "compress_kv", "kv_capacity"]


STATS_HEAD = 16  # tau, g, mstar, R_K, R_Q, T0, nblocks, ncand, Fread, Fdot, 0 x 6; then kbar[d]


def STATS_STRIDE(d: int) -> int:
    return STATS_HEAD + d


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise WildcatError("WildCat runs on CUDA tensors only (no CPU fallback)")


def _cont(t):
    return None if t is None else t.contiguous()


@dataclass
class Selection:
    S: torch.Tensor       # int32 [units, r]
    r_eff: torch.Tensor   # int32 [units]
    L: torch.Tensor       # float64 [units, r, r]
    stats: torch.Tensor   # float64 [units, 16 + d]: tau, g, mstar, R_K, R_Q, T0, nblocks, ncand, Fread, ..., kbar
    shape: B.wc_shape
    opts: B.wc_opts


@dataclass
class Cache:
    KS: torch.Tensor      # dtype [units, r, d]
    X: torch.Tensor       # float32 [units, r, d+1] = [V_S, w]
    vmin: torch.Tensor    # dtype [units, d]
    vmax: torch.Tensor
    r_eff: torch.Tensor
    heads_kv: int
    opts: B.wc_opts
    shape: B.wc_shape = None  # the selection's shape (n, r, bins)


@dataclass
class KvCache:
    """Compact KV cache of compress_kv (reading Z24): per unit C rows of a key, a value (model dtype)
    and a weight (fp32); rows [0, c_eff) valid."""
    KC: torch.Tensor      # dtype [units, C, d]
    VC: torch.Tensor      # dtype [units, C, d]
    WC: torch.Tensor      # float32 [units, C]
    vmin: torch.Tensor    # dtype [units, d]
    vmax: torch.Tensor
    r_eff: torch.Tensor   # int32 [units]: c_eff
    heads_kv: int
    opts: B.wc_opts
    n: int = 0            # context length the cache was built from

    @property
    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.KC, self.VC, self.WC))


_ws_cache: dict = {}


def _stream_of(stream):
    return torch.cuda.current_stream() if stream is None else stream


def _workspace(shape, op, device, stream=None, nbytes=None):
    """Scratch for one call, cached per (device, op, stream): calls on one stream are serialised by
    the stream, so they may share it; another stream gets its own buffer.  A buffer allocated while a
    different stream is current is tied to the launching stream with record_stream, so the caching
    allocator never hands its memory out while the library's kernels still use it."""
    nb = B.workspace_bytes(shape, op) if nbytes is None else nbytes
    st = _stream_of(stream)
    key = (device, op, st.cuda_stream)
    t = _ws_cache.get(key)
    if t is None or t.numel() < nb:
        t = torch.empty(max(nb, 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = t
        _on_stream(st, t)
    return t


def _on_stream(stream, *ts):
    """Outputs allocated on the current stream but written on `stream`: record the use."""
    if stream is None or stream == torch.cuda.current_stream():
        return
    for t in ts:
        if t is not None:
            t.record_stream(stream)


def _opts(seed, beta, rq, clip, block, kw):
    """wc_opts from the common keywords plus the optional ones: unit_offset (PAR2: global id of unit 0),
    tau_one (WC_TAU_ONE), recenter (False -> WC_NO_RECENTER), check_finite (WC_CHECK_FINITE)."""
    bad = set(kw) - {"unit_offset", "tau_one", "recenter", "check_finite"}
    if bad:
        raise TypeError(f"unexpected keyword arguments {sorted(bad)}")
    return B.make_opts(seed, beta, rq, clip, block=block, **kw)


def select(Q, K, r, seed=0, beta=None, rq=None, block=1, bins=1, stream=None, **kw) -> Selection:
    """RPNys selection; block >= 2 selects the blocked (accelerated) variant (reading Z22); bins > 1
    runs Alg 2 binning (S [units][R] concatenated over bins, L [units*B][rb][rb], stats per bin).
    Keywords unit_offset / tau_one / recenter / check_finite: see _opts."""
    Q, K = _cont(Q), _cont(K)
    _require_cuda(Q, K)
    shape = B.make_shape(Q, K, r, bins=bins)
    opts = _opts(seed, beta, rq, True, block, kw)
    units = shape.batch * shape.heads_kv
    rb, R = B.coreset_rows(shape.n, r, bins)
    dev = K.device
    S = torch.empty(units, R, dtype=torch.int32, device=dev)
    reff = torch.empty(units, dtype=torch.int32, device=dev)
    L = torch.empty(units * bins, rb, rb, dtype=torch.float64, device=dev)
    stats = torch.empty(units * bins, STATS_STRIDE(shape.d), dtype=torch.float64, device=dev)
    ws = _workspace(shape, B.WC_OP_SELECT, dev, stream)
    _on_stream(stream, S, reff, L, stats)
    B.wildcat_select(shape, opts, Q, K, S, reff, L, stats, ws, stream)
    return Selection(S, reff, L, stats, shape, opts)


def weights(K, V, sel: Selection, stream=None) -> Cache:
    K, V = _cont(K), _cont(V)
    _require_cuda(K, V)
    shape = sel.shape
    units, d = shape.batch * shape.heads_kv, shape.d
    _, R = B.coreset_rows(shape.n, shape.r, shape.bins)
    dev = K.device
    KS = torch.empty(units, R, d, dtype=K.dtype, device=dev)
    X = torch.empty(units, R, d + 1, dtype=torch.float32, device=dev)
    vmin = torch.empty(units, d, dtype=K.dtype, device=dev)
    vmax = torch.empty(units, d, dtype=K.dtype, device=dev)
    ws = _workspace(shape, B.WC_OP_WEIGHTS, dev, stream)
    _on_stream(stream, KS, X, vmin, vmax)
    B.wildcat_weights(shape, sel.opts, K, V, sel.S, sel.r_eff, sel.L, sel.stats, KS, X, vmin, vmax, ws, stream)
    return Cache(KS, X, vmin, vmax, sel.r_eff, shape.heads_kv, sel.opts, shape)


def attend(Q, cache, beta=None, clip=None, stream=None):
    """Alg 3 WtdAttn of Q over a Cache (weights()) or a compact KvCache (compress_kv: wildcat_decode)."""
    Q = _cont(Q)
    _require_cuda(Q)
    if isinstance(cache, KvCache):
        return decode(Q, cache, beta=beta, clip=clip, stream=stream)
    b, hq, m, d = Q.shape
    units, r, _ = cache.KS.shape
    if cache.shape is not None:  # the selection's (n, r, bins) define the coreset layout
        cs = cache.shape
        shape = B.wc_shape(batch=b, heads_q=hq, heads_kv=cache.heads_kv, d=d, r=cs.r, bins=cs.bins,
                           dtype=B._dtype_code(Q), reserved=0, m=m, n=cs.n)
    else:
        shape = B.wc_shape(batch=b, heads_q=hq, heads_kv=cache.heads_kv, d=d, r=r, bins=1,
                           dtype=B._dtype_code(Q), reserved=0, m=m, n=max(r, 1))
    flags = cache.opts.flags if clip is None else ((cache.opts.flags & ~B.WC_NO_CLIP) | (0 if clip else B.WC_NO_CLIP))
    opts = B.wc_opts(beta=cache.opts.beta if beta is None else float(beta), rq=cache.opts.rq,
                     seed=cache.opts.seed, flags=flags, block=0, unit_offset=cache.opts.unit_offset)
    O = torch.empty_like(Q)
    ws = _workspace(shape, B.WC_OP_ATTEND, Q.device, stream) if B.workspace_bytes(shape, B.WC_OP_ATTEND) else None
    _on_stream(stream, O)
    B.wildcat_attend(shape, opts, Q, cache.KS, cache.X, cache.r_eff, cache.vmin, cache.vmax, O, ws, stream)
    return O


def forward(Q, K, V, r, seed=0, beta=None, rq=None, clip=True, out=None, S=None, r_eff=None, block=1,
            bins=1, stream=None, **kw):
    """Alg 4 WildCat on device tensors.  Returns O (and fills S [units][R] / r_eff if given).
    block >= 2: blocked (accelerated) RPCholesky selection with b = block (reading Z22).
    bins > 1: Alg 2 binning with B = bins (R = B * min(ceil(r/B), n/B) coreset rows per unit).
    unit_offset = u0: these units are units [u0, u0 + units) of a larger batch (PAR2 partition: the
    same pivots as the one-GPU run); tau_one / recenter / check_finite: see _opts."""
    Q, K, V = _cont(Q), _cont(K), _cont(V)
    _require_cuda(Q, K, V)
    shape = B.make_shape(Q, K, r, bins=bins)
    opts = _opts(seed, beta, rq, clip, block, kw)
    O = torch.empty_like(Q) if out is None else out
    ws = _workspace(shape, B.WC_OP_FORWARD, K.device, stream)
    if out is None:
        _on_stream(stream, O)
    B.wildcat_forward(shape, opts, Q, K, V, O, S, r_eff, ws, stream)
    return O


def decode(Q, cache: KvCache, beta=None, clip=None, stream=None):
    """WtdAttn of Q [batch, hq, m, d] (new queries) over a compact KV cache (wildcat_decode)."""
    Q = _cont(Q)
    _require_cuda(Q)
    b, hq, m, d = Q.shape
    units, C, _ = cache.KC.shape
    shape = B.wc_shape(batch=b, heads_q=hq, heads_kv=cache.heads_kv, d=d, r=C, bins=1, dtype=B._dtype_code(Q),
                       reserved=0, m=m, n=max(C, cache.n))
    flags = cache.opts.flags if clip is None else ((cache.opts.flags & ~B.WC_NO_CLIP) | (0 if clip else B.WC_NO_CLIP))
    opts = B.wc_opts(beta=cache.opts.beta if beta is None else float(beta), rq=cache.opts.rq, seed=cache.opts.seed,
                     flags=flags, block=0, unit_offset=cache.opts.unit_offset)
    O = torch.empty_like(Q)
    nb = B.decode_workspace_bytes(shape)
    ws = _workspace(shape, "decode", Q.device, stream, nbytes=nb) if nb else None
    _on_stream(stream, O)
    B.wildcat_decode(shape, opts, Q, cache.KC, cache.VC, cache.WC, cache.r_eff, cache.vmin, cache.vmax, O, ws, stream)
    return O


def kv_capacity(n, r, keep_first=0, keep_last=0, bins=1) -> int:
    """Cache rows per unit of compress_kv: keep_first + keep_last + B * min(ceil(r/B), n_mid/B)."""
    nmid = int(n) - int(keep_first) - int(keep_last)
    return int(keep_first) + int(keep_last) + (B.coreset_rows(nmid, r, bins)[1] if nmid > 0 else 0)


def compress_kv(Q, K, V, r, keep_first=0, keep_last=0, bins=1, seed=0, beta=None, rq=None, block=1, S=None,
                stream=None, **kw) -> KvCache:
    """KV-cache compression (E3 protocol P:667-669; reading Z24): the first keep_first and
    last keep_last tokens of every (batch, kv-head) are kept exactly, the middle goes through
    CompressKV (Alg 2) at rank r with `bins` bins.  Q holds the prompt's queries (for R_Q) or may be
    None when rq is given.  Returns a compact KvCache whose rows are [retained | coreset | zero]
    (r_eff = c_eff), ready for attend(Q_new, cache) -- the decode step.  S (int32 [units][R]), if given,
    receives the global token index of each coreset row."""
    Q, K, V = _cont(Q), _cont(K), _cont(V)
    _require_cuda(Q, K, V)
    if Q is None and rq is None:
        raise WildcatError("compress_kv needs the prompt queries Q or rq")
    b, hkv, n, d = K.shape
    shape = B.make_shape(Q, K, r, bins=bins)
    opts = _opts(seed, beta, rq, True, block, kw)
    C = B.kv_capacity(shape, keep_first, keep_last)
    if C == 0:
        raise WildcatError("compress_kv: invalid split (keep_first/keep_last/r/bins)")
    units, dev = b * hkv, K.device
    KC = torch.empty(units, C, d, dtype=K.dtype, device=dev)
    VC = torch.empty(units, C, d, dtype=K.dtype, device=dev)
    WC = torch.empty(units, C, dtype=torch.float32, device=dev)
    ceff = torch.empty(units, dtype=torch.int32, device=dev)
    vmin = torch.empty(units, d, dtype=K.dtype, device=dev)
    vmax = torch.empty(units, d, dtype=K.dtype, device=dev)
    ws = _workspace(shape, "kv", dev, stream, nbytes=B.kv_workspace_bytes(shape, keep_first, keep_last))
    _on_stream(stream, KC, VC, WC, ceff, vmin, vmax)
    B.wildcat_compress_kv(shape, opts, keep_first, keep_last, Q, K, V, KC, VC, WC, ceff, vmin, vmax, S, ws, stream)
    return KvCache(KC, VC, WC, vmin, vmax, ceff, hkv, opts, n)


class HostForward:
    """End-to-end WildCat on host (CPU) buffers with persistent device buffers.

    Per call: H2D of K and Q, wildcat_select, then wildcat_weights once the H2D of V (issued on a
    side stream after K and Q, so it overlaps the selection) has landed, wildcat_attend, D2H of O
    into a pinned buffer, synchronise.  Every step is a C-ABI call (include/wildcat.h)."""

    def __init__(self, Q, K, r, seed=0, beta=None, rq=None, clip=True, block=1, bins=1, device="cuda", **kw):
        dev = torch.device(device)
        self.dev, self.r = dev, int(r)
        self.Qd = torch.empty(Q.shape, dtype=Q.dtype, device=dev)
        self.Kd = torch.empty(K.shape, dtype=K.dtype, device=dev)
        self.Vd = torch.empty(K.shape, dtype=K.dtype, device=dev)
        self.Od = torch.empty(Q.shape, dtype=Q.dtype, device=dev)
        self.Oh = torch.empty(Q.shape, dtype=Q.dtype, pin_memory=True)
        self.shape = B.make_shape(self.Qd, self.Kd, r, bins=bins)
        self.opts = _opts(seed, beta, rq, clip, block, kw)
        units, d = self.shape.batch * self.shape.heads_kv, self.shape.d
        rb, R = B.coreset_rows(self.shape.n, r, bins)
        self.S = torch.empty(units, R, dtype=torch.int32, device=dev)
        self.reff = torch.empty(units, dtype=torch.int32, device=dev)
        self.L = torch.empty(units * bins, rb, rb, dtype=torch.float64, device=dev)
        self.stats = torch.empty(units * bins, STATS_STRIDE(d), dtype=torch.float64, device=dev)
        self.KS = torch.empty(units, R, d, dtype=K.dtype, device=dev)
        self.X = torch.empty(units, R, d + 1, dtype=torch.float32, device=dev)
        self.vmin = torch.empty(units, d, dtype=K.dtype, device=dev)
        self.vmax = torch.empty(units, d, dtype=K.dtype, device=dev)
        self.ws_s = B.alloc_workspace(self.shape, B.WC_OP_SELECT, dev)
        self.ws_w = B.alloc_workspace(self.shape, B.WC_OP_WEIGHTS, dev)
        na = B.workspace_bytes(self.shape, B.WC_OP_ATTEND)
        self.ws_a = B.alloc_workspace(self.shape, B.WC_OP_ATTEND, dev) if na else None
        self.s_main = torch.cuda.Stream(dev)
        self.s_v = torch.cuda.Stream(dev)
        self.ev_kq = torch.cuda.Event()
        self.ev_v = torch.cuda.Event()

    def __call__(self, Qh, Kh, Vh, out=None):
        """Returns O on the host.  With out=None a fresh tensor (a copy of the persistent pinned
        buffer, so earlier results are never overwritten); with out= (a host tensor of Q's shape and
        dtype, ideally pinned) O is written there directly and `out` is returned."""
        if out is not None and (out.shape != self.Oh.shape or out.dtype != self.Oh.dtype or out.is_cuda):
            raise WildcatError("forward_host: out must be a host tensor of Q's shape and dtype")
        sm, sv = self.s_main, self.s_v
        with torch.cuda.stream(sm):
            self.Kd.copy_(Kh, non_blocking=True)
            self.Qd.copy_(Qh, non_blocking=True)
            self.ev_kq.record(sm)
        with torch.cuda.stream(sv):
            sv.wait_event(self.ev_kq)  # V after K and Q on the link, overlapping the selection
            self.Vd.copy_(Vh, non_blocking=True)
            self.ev_v.record(sv)
        B.wildcat_select(self.shape, self.opts, self.Qd, self.Kd, self.S, self.reff, self.L, self.stats, self.ws_s, sm)
        sm.wait_event(self.ev_v)
        B.wildcat_weights(self.shape, self.opts, self.Kd, self.Vd, self.S, self.reff, self.L, self.stats, self.KS,
                          self.X, self.vmin, self.vmax, self.ws_w, sm)
        B.wildcat_attend(self.shape, self.opts, self.Qd, self.KS, self.X, self.reff, self.vmin, self.vmax, self.Od,
                         self.ws_a, sm)
        dst = self.Oh if out is None else out
        with torch.cuda.stream(sm):
            dst.copy_(self.Od, non_blocking=True)
        sm.synchronize()
        return self.Oh.clone() if out is None else out


class HostPipeline:
    """Streaming end-to-end WildCat over a sequence of host (CPU, pinned) batches of one shape.

    Each submitted step copies its Q, K, V host->device, runs wildcat_forward (the fused C-ABI
    call) and copies O device->host into the caller's pinned `out`.  The three parts run on three
    CUDA streams ordered by events over `slots` device buffer sets, so the H2D of step k+1 and
    the D2H of step k-1 overlap the compute of step k (B200: the copy engines of both directions and
    the SMs work at once; one compute stream keeps the compute serial and its workspace shared).
        pipe = HostPipeline(Q, K, r, block=16)
        for Qh, Kh, Vh, Oh in batches: pipe.submit(Qh, Kh, Vh, Oh)
        pipe.synchronize()            # every Oh holds its step's result
    A step's `out` may be read once pipe.done(step) (or synchronize()) returns; its inputs may be
    overwritten once pipe.inputs_free(step) does."""

    def __init__(self, Q, K, r, seed=0, beta=None, rq=None, clip=True, block=1, bins=1, device="cuda", slots=2,
                 **kw):
        dev = torch.device(device)
        self.dev, self.nslots = dev, int(slots)
        mk = lambda t: torch.empty(t.shape, dtype=t.dtype, device=dev)  # noqa: E731
        self.buf = [dict(Q=mk(Q), K=mk(K), V=mk(K), O=mk(Q)) for _ in range(self.nslots)]
        self.shape = B.make_shape(self.buf[0]["Q"], self.buf[0]["K"], r, bins=bins)
        self.opts = _opts(seed, beta, rq, clip, block, kw)
        self.ws = B.alloc_workspace(self.shape, B.WC_OP_FORWARD, dev)
        self.s_in, self.s_cmp, self.s_out = (torch.cuda.Stream(dev) for _ in range(3))
        self.ev_in = [torch.cuda.Event() for _ in range(self.nslots)]
        self.ev_cmp = [torch.cuda.Event() for _ in range(self.nslots)]
        self.ev_out = [torch.cuda.Event() for _ in range(self.nslots)]
        self.step = 0

    def submit(self, Qh, Kh, Vh, out):
        """Enqueue one step (host tensors; pinned for asynchronous copies).  Returns its index."""
        for t, ref in ((Qh, "Q"), (Kh, "K"), (Vh, "V"), (out, "O")):
            want = self.buf[0][ref]
            if t.is_cuda or t.shape != want.shape or t.dtype != want.dtype:
                raise WildcatError(f"HostPipeline.submit: {ref} must be a host tensor of shape {tuple(want.shape)}")
        k, s = self.step, self.step % self.nslots
        b = self.buf[s]
        with torch.cuda.stream(self.s_in):
            if k >= self.nslots:  # the compute of step k - slots has read this slot's inputs
                self.s_in.wait_event(self.ev_cmp[s])
            b["K"].copy_(Kh, non_blocking=True)
            b["Q"].copy_(Qh, non_blocking=True)
            b["V"].copy_(Vh, non_blocking=True)
            self.ev_in[s].record(self.s_in)
        self.s_cmp.wait_event(self.ev_in[s])
        if k >= self.nslots:  # the D2H of step k - slots has read this slot's output
            self.s_cmp.wait_event(self.ev_out[s])
        B.wildcat_forward(self.shape, self.opts, b["Q"], b["K"], b["V"], b["O"], None, None, self.ws, self.s_cmp)
        self.ev_cmp[s].record(self.s_cmp)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_cmp[s])
            out.copy_(b["O"], non_blocking=True)
            self.ev_out[s].record(self.s_out)
        self.step += 1
        return k

    def done(self, k):
        """Block until step k's result is in its host `out` (valid for the last `slots` steps)."""
        self.ev_out[k % self.nslots].synchronize()

    def inputs_free(self, k):
        """Block until step k's host inputs have been copied (they may then be overwritten)."""
        self.ev_in[k % self.nslots].synchronize()

    def synchronize(self):
        for st in (self.s_in, self.s_cmp, self.s_out):
            st.synchronize()


_host_cache: dict = {}


def forward_host(Q, K, V, r, seed=0, beta=None, rq=None, clip=True, device="cuda", block=1, bins=1, out=None, **kw):
    """End-to-end call with host (CPU) buffers: H2D copies, the CUDA path, D2H copy of O (into `out`
    if given, else into a new host tensor).  Device buffers persist per (shapes, options); see
    HostForward.  Calls with the same key share those device buffers: serialise them."""
    key = (tuple(Q.shape), tuple(K.shape), Q.dtype, int(r), seed, beta, rq, clip, int(block), int(bins), str(device),
           tuple(sorted(kw.items())))
    hf = _host_cache.get(key)
    if hf is None:
        hf = HostForward(Q, K, r, seed=seed, beta=beta, rq=rq, clip=clip, block=block, bins=bins, device=device, **kw)
        _host_cache[key] = hf
    return hf(Q, K, V, out=out)


# --------------------------------------------------------------------------- n-sharded (PAR3)
def shard_range(n_global: int, world: int, rank: int):
    """Contiguous key shard of `rank`: sizes differ by at most one, every rank non-empty."""
    if not 1 <= world <= n_global:
        raise WildcatError("need 1 <= world <= n_global")
    base, extra = divmod(n_global, world)
    off = rank * base + min(rank, extra)
    return off, base + (1 if rank < extra else 0)


class NshardComm:
    """NCCL communicator owned by libwildcat (one per process / GPU)."""

    def __init__(self, handle, world: int, rank: int):
        self.handle, self.world, self.rank = handle, world, rank

    @classmethod
    def create(cls, world: int | None = None, rank: int | None = None, group=None, transport: str = "nccl",
               capacity: int = 1 << 18):
        """transport "nccl": NCCL collectives per exchange; "p2p": device-initiated peer-memory
        mailboxes (CUDA IPC; handles exchanged over `group`, which may be a gloo group)."""
        import torch.distributed as dist

        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        if transport == "p2p":
            h, mine = B.wc_p2p_comm_create(world, rank, capacity)
            if world > 1:
                allh = [None] * world
                dist.all_gather_object(allh, mine, group=group)
                B.wc_p2p_comm_connect(h, allh)
            return cls(h, world, rank)
        if transport != "nccl":
            raise WildcatError(f"unknown transport {transport!r}")
        uid = [B.wc_comm_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0, group=group)
        return cls(B.wc_comm_init(uid[0], world, rank), world, rank)

    def close(self):
        if self.handle is not None:
            B.wc_comm_destroy(self.handle)
            self.handle = None


def forward_nshard(comm: NshardComm, Q, K, V, r, n_global, n_offset, seed=0, beta=None, rq=None, clip=True,
                   S=None, r_eff=None, out=None, stream=None, block=1, **kw):
    """Alg 4 for one (batch, kv-head) unit whose keys are sharded over the communicator's ranks.
    K, V: this rank's [1, 1, n_local, d] shard at global offset n_offset; Q: [1, hq, m_local, d].
    block >= 2 (<= 16): blocked selection (reading Z22), one candidate exchange per block."""
    Q, K, V = _cont(Q), _cont(K), _cont(V)
    _require_cuda(Q, K, V)
    shape = B.make_shape(Q, K, r)
    opts = _opts(seed, beta, rq, clip, block, kw)
    O = torch.empty_like(Q) if out is None else out
    ws = _workspace(shape, B.WC_OP_FORWARD_NSHARD, K.device, stream)
    if out is None:
        _on_stream(stream, O)
    B.wildcat_forward_nshard(comm.handle, shape, n_global, n_offset, opts, Q, K, V, O, S, r_eff, ws, stream)
    return O
