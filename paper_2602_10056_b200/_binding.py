"""ctypes binding of libwildcat.so -- argument marshalling only.

Every function here has the name of the C entry point it wraps (include/wildcat.h)
and does nothing but turn torch tensors into pointers and sizes.  All arithmetic of
the method runs in the CUDA kernels behind the C ABI.  There is no CPU fallback:
if the shared library is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwildcat.so")

WC_F32, WC_BF16 = 0, 1
WC_OP_SELECT, WC_OP_WEIGHTS, WC_OP_ATTEND, WC_OP_FORWARD, WC_OP_FORWARD_NSHARD = 0, 1, 2, 3, 4
WC_NO_CLIP, WC_TAU_ONE, WC_NO_RECENTER, WC_CHECK_FINITE = 1, 2, 4, 8
WC_ENONFINITE = -8


class WildcatError(RuntimeError):
    pass


class wc_shape(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("heads_q", ctypes.c_int32), ("heads_kv", ctypes.c_int32),
                ("d", ctypes.c_int32), ("r", ctypes.c_int32), ("bins", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("m", ctypes.c_int64), ("n", ctypes.c_int64)]


class wc_opts(ctypes.Structure):
    _fields_ = [("beta", ctypes.c_double), ("rq", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("flags", ctypes.c_uint32), ("block", ctypes.c_uint32), ("unit_offset", ctypes.c_uint64)]


_lib = None


def lib():
    """Load libwildcat.so (building it first if the sources are newer).  Raises if unavailable."""
    global _lib
    if _lib is None:
        from . import build as _build

        try:
            _build.build()
        except Exception as e:  # nvcc missing on the box: use the shipped .so if present
            if not os.path.exists(LIB_PATH):
                raise WildcatError(f"libwildcat.so is missing and could not be built: {e}") from e
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        S = ctypes.POINTER(wc_shape)
        O = ctypes.POINTER(wc_opts)
        L.wc_workspace_bytes.argtypes = [S, ctypes.c_int]
        L.wc_workspace_bytes.restype = ctypes.c_size_t
        L.wildcat_select.argtypes = [S, O, P, P, P, P, P, P, P, ctypes.c_size_t, P]
        L.wildcat_weights.argtypes = [S, O, P, P, P, P, P, P, P, P, P, P, P, ctypes.c_size_t, P]
        L.wildcat_attend.argtypes = [S, O, P, P, P, P, P, P, P, P, ctypes.c_size_t, P]
        L.wildcat_forward.argtypes = [S, O, P, P, P, P, P, P, P, ctypes.c_size_t, P]
        for f in ("wildcat_select", "wildcat_weights", "wildcat_attend", "wildcat_forward"):
            getattr(L, f).restype = ctypes.c_int
        L.wc_strerror.argtypes = [ctypes.c_int]
        L.wc_strerror.restype = ctypes.c_char_p
        L.wc_last_launch_count.restype = ctypes.c_int
        L.wc_version.restype = ctypes.c_int
        L.wc_comm_unique_id.argtypes = [P]
        L.wc_comm_init.argtypes = [ctypes.POINTER(ctypes.c_void_p), P, ctypes.c_int, ctypes.c_int]
        L.wc_comm_destroy.argtypes = [P]
        L.wildcat_forward_nshard.argtypes = [P, S, ctypes.c_int64, ctypes.c_int64, O, P, P, P, P, P, P, P,
                                             ctypes.c_size_t, P]
        L.wc_p2p_comm_create.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int, ctypes.c_size_t, P]
        L.wc_p2p_comm_connect.argtypes = [P, P]
        for f in ("wc_comm_unique_id", "wc_comm_init", "wc_comm_destroy", "wildcat_forward_nshard",
                  "wc_p2p_comm_create", "wc_p2p_comm_connect"):
            getattr(L, f).restype = ctypes.c_int
        L.wc_kv_capacity.argtypes = [S, ctypes.c_int32, ctypes.c_int32]
        L.wc_kv_capacity.restype = ctypes.c_size_t
        L.wc_kv_workspace_bytes.argtypes = [S, ctypes.c_int32, ctypes.c_int32]
        L.wc_kv_workspace_bytes.restype = ctypes.c_size_t
        L.wildcat_compress_kv.argtypes = [S, O, ctypes.c_int32, ctypes.c_int32, P, P, P, P, P, P, P, P, P, P, P,
                                          ctypes.c_size_t, P]
        L.wildcat_compress_kv.restype = ctypes.c_int
        L.wc_decode_workspace_bytes.argtypes = [S]
        L.wc_decode_workspace_bytes.restype = ctypes.c_size_t
        L.wildcat_decode.argtypes = [S, O, P, P, P, P, P, P, P, P, P, ctypes.c_size_t, P]
        L.wildcat_decode.restype = ctypes.c_int
        L.wc_timing_enable.argtypes = [ctypes.c_int]
        L.wc_timing_enable.restype = ctypes.c_int
        L.wc_timing_read.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_int]
        L.wc_timing_read.restype = ctypes.c_int
        _lib = L
    return _lib


class NonFiniteInput(WildcatError):
    """WC_CHECK_FINITE found a NaN or Inf in an input."""


def _check(rc: int, what: str) -> None:
    if rc == WC_ENONFINITE:
        raise NonFiniteInput(f"{what}: {lib().wc_strerror(rc).decode()} ({rc})")
    if rc != 0:
        raise WildcatError(f"{what}: {lib().wc_strerror(rc).decode()} ({rc})")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return WC_F32
    if t.dtype == torch.bfloat16:
        return WC_BF16
    raise WildcatError(f"unsupported dtype {t.dtype}")


def make_shape(Q, K, r, m=None, bins=1) -> wc_shape:
    b, hkv, n, d = K.shape
    hq = Q.shape[1] if Q is not None else hkv
    mm = (Q.shape[2] if Q is not None else 0) if m is None else m
    return wc_shape(batch=b, heads_q=hq, heads_kv=hkv, d=d, r=int(r), bins=int(bins), dtype=_dtype_code(K),
                    reserved=0, m=mm, n=n)


def coreset_rows(n: int, r: int, bins: int = 1):
    """(rb, R): per-bin rank min(ceil(r/B), n/B) and coreset rows B*rb per unit (Z13; R = r if B = 1)."""
    rb = min(-(-int(r) // int(bins)), int(n) // int(bins))
    return rb, int(bins) * rb


def make_opts(seed=0, beta=None, rq=None, clip=True, block=1, unit_offset=0, tau_one=False, recenter=True,
              check_finite=False) -> wc_opts:
    """wc_opts: unit_offset = global id of the call's unit 0 (PAR2 partitions); tau_one -> WC_TAU_ONE;
    recenter=False -> WC_NO_RECENTER; check_finite -> WC_CHECK_FINITE (include/wildcat.h)."""
    flags = ((0 if clip else WC_NO_CLIP) | (WC_TAU_ONE if tau_one else 0) | (0 if recenter else WC_NO_RECENTER)
             | (WC_CHECK_FINITE if check_finite else 0))
    return wc_opts(beta=-1.0 if beta is None else float(beta), rq=-1.0 if rq is None else float(rq),
                   seed=int(seed) & 0xFFFFFFFFFFFFFFFF, flags=flags, block=int(block),
                   unit_offset=int(unit_offset))


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def workspace_bytes(shape: wc_shape, op: int) -> int:
    return int(lib().wc_workspace_bytes(ctypes.byref(shape), op))


def alloc_workspace(shape: wc_shape, op: int, device) -> torch.Tensor:
    nb = workspace_bytes(shape, op)
    return torch.empty(max(nb, 256), dtype=torch.uint8, device=device)


# ---- argument checks (before any ctypes call): the C ABI takes raw pointers, so a tensor that
# disagrees with the shape would be read or written out of bounds.  Every wrapper checks dtype,
# device, contiguity and size of each tensor against the wc_shape it passes.
_TDT = {WC_F32: torch.float32, WC_BF16: torch.bfloat16}


def _need(t, name, dtype, numel, device=None, exact=False, optional=False):
    if t is None:
        if optional:
            return None
        raise WildcatError(f"{name}: tensor required")
    if not isinstance(t, torch.Tensor):
        raise WildcatError(f"{name}: expected a torch.Tensor")
    if not t.is_cuda:
        raise WildcatError(f"{name}: must be a CUDA tensor (no CPU fallback)")
    if device is not None and t.device != device:
        raise WildcatError(f"{name}: on {t.device}, expected {device}")
    if not t.is_contiguous():
        raise WildcatError(f"{name}: must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise WildcatError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if (t.numel() != numel) if exact else (t.numel() < numel):
        raise WildcatError(f"{name}: {t.numel()} elements, expected {'' if exact else '>= '}{numel}")
    return t.device


def _dims(shape):
    units = shape.batch * shape.heads_kv
    rb, R = coreset_rows(shape.n, shape.r, shape.bins)
    return units, rb, R, shape.d, _TDT.get(shape.dtype)


def _check_sel_out(shape, dev, S, r_eff, L, stats, optional_S=False):
    units, rb, R, d, _ = _dims(shape)
    _need(S, "S", torch.int32, units * R, dev, optional=optional_S)
    _need(r_eff, "r_eff", torch.int32, units, dev, optional=optional_S)
    if L is not None or stats is not None:
        _need(L, "L", torch.float64, units * shape.bins * rb * rb, dev)
        _need(stats, "stats", torch.float64, units * shape.bins * (16 + d), dev)


def _check_qkv(shape, Q, K, V=None, O=None, q_optional=False, need_v=False, need_o=False):
    units, _, _, d, tdt = _dims(shape)
    dev = _need(K, "K", tdt, units * shape.n * d, exact=True)
    _need(V, "V", tdt, units * shape.n * d, dev, exact=True, optional=not need_v)
    nq = shape.batch * shape.heads_q * shape.m * d
    _need(Q, "Q", tdt, nq, dev, exact=True, optional=q_optional or nq == 0)
    _need(O, "O", tdt, nq, dev, exact=True, optional=not need_o or nq == 0)
    return dev


def _check_ws(ws, dev, op_bytes):
    if op_bytes:
        _need(ws, "workspace", torch.uint8, op_bytes, dev)


def wildcat_select(shape, opts, Q, K, S, r_eff, L, stats, ws, stream=None):
    dev = _check_qkv(shape, Q, K, q_optional=opts.rq >= 0)
    _check_sel_out(shape, dev, S, r_eff, L, stats)
    _check_ws(ws, dev, workspace_bytes(shape, WC_OP_SELECT))
    rc = lib().wildcat_select(ctypes.byref(shape), ctypes.byref(opts), _ptr(Q), _ptr(K), _ptr(S), _ptr(r_eff),
                              _ptr(L), _ptr(stats), _ptr(ws), ws.numel(), _stream(stream))
    _check(rc, "wildcat_select")


def wildcat_weights(shape, opts, K, V, S, r_eff, L, stats, KS, X, vmin, vmax, ws, stream=None):
    units, rb, R, d, tdt = _dims(shape)
    dev = _check_qkv(shape, None, K, V, q_optional=True, need_v=True)
    _check_sel_out(shape, dev, S, r_eff, L, stats)
    _need(KS, "KS", tdt, units * R * d, dev)
    _need(X, "X", torch.float32, units * R * (d + 1), dev)
    _need(vmin, "vmin", tdt, units * d, dev)
    _need(vmax, "vmax", tdt, units * d, dev)
    _check_ws(ws, dev, workspace_bytes(shape, WC_OP_WEIGHTS))
    rc = lib().wildcat_weights(ctypes.byref(shape), ctypes.byref(opts), _ptr(K), _ptr(V), _ptr(S), _ptr(r_eff),
                               _ptr(L), _ptr(stats), _ptr(KS), _ptr(X), _ptr(vmin), _ptr(vmax), _ptr(ws),
                               ws.numel(), _stream(stream))
    _check(rc, "wildcat_weights")


def wildcat_attend(shape, opts, Q, KS, X, r_eff, vmin, vmax, O, ws=None, stream=None):
    units, _, R, d, tdt = _dims(shape)
    nq = shape.batch * shape.heads_q * shape.m * d
    dev = _need(KS, "KS", tdt, units * R * d)
    _need(Q, "Q", tdt, nq, dev, exact=True, optional=nq == 0)
    _need(O, "O", tdt, nq, dev, exact=True, optional=nq == 0)
    _need(X, "X", torch.float32, units * R * (d + 1), dev)
    _need(r_eff, "r_eff", torch.int32, units, dev)
    _need(vmin, "vmin", tdt, units * d, dev)
    _need(vmax, "vmax", tdt, units * d, dev)
    _check_ws(ws, dev, workspace_bytes(shape, WC_OP_ATTEND))
    rc = lib().wildcat_attend(ctypes.byref(shape), ctypes.byref(opts), _ptr(Q), _ptr(KS), _ptr(X), _ptr(r_eff),
                              _ptr(vmin), _ptr(vmax), _ptr(O), _ptr(ws), 0 if ws is None else ws.numel(),
                              _stream(stream))
    _check(rc, "wildcat_attend")


def wildcat_forward(shape, opts, Q, K, V, O, S, r_eff, ws, stream=None):
    dev = _check_qkv(shape, Q, K, V, O, need_v=True, need_o=True)
    _check_sel_out(shape, dev, S, r_eff, None, None, optional_S=True)
    _check_ws(ws, dev, workspace_bytes(shape, WC_OP_FORWARD))
    rc = lib().wildcat_forward(ctypes.byref(shape), ctypes.byref(opts), _ptr(Q), _ptr(K), _ptr(V), _ptr(O),
                               _ptr(S), _ptr(r_eff), _ptr(ws), ws.numel(), _stream(stream))
    _check(rc, "wildcat_forward")


def kv_capacity(shape, keep_first, keep_last) -> int:
    return int(lib().wc_kv_capacity(ctypes.byref(shape), int(keep_first), int(keep_last)))


def kv_workspace_bytes(shape, keep_first, keep_last) -> int:
    return int(lib().wc_kv_workspace_bytes(ctypes.byref(shape), int(keep_first), int(keep_last)))


def wildcat_compress_kv(shape, opts, keep_first, keep_last, Q, K, V, KC, VC, WC, c_eff, vmin, vmax, S, ws,
                        stream=None):
    units, _, _, d, tdt = _dims(shape)
    C = kv_capacity(shape, keep_first, keep_last)
    if C == 0:
        raise WildcatError("wildcat_compress_kv: invalid split (keep_first / keep_last / r / bins)")
    dev = _check_qkv(shape, Q, K, V, q_optional=True, need_v=True)
    _need(KC, "KC", tdt, units * C * d, dev)
    _need(VC, "VC", tdt, units * C * d, dev)
    _need(WC, "WC", torch.float32, units * C, dev)
    _need(c_eff, "c_eff", torch.int32, units, dev)
    _need(vmin, "vmin", tdt, units * d, dev)
    _need(vmax, "vmax", tdt, units * d, dev)
    _need(S, "S", torch.int32, units * (C - int(keep_first) - int(keep_last)), dev, optional=True)
    _check_ws(ws, dev, kv_workspace_bytes(shape, keep_first, keep_last))
    rc = lib().wildcat_compress_kv(ctypes.byref(shape), ctypes.byref(opts), int(keep_first), int(keep_last), _ptr(Q),
                                   _ptr(K), _ptr(V), _ptr(KC), _ptr(VC), _ptr(WC), _ptr(c_eff), _ptr(vmin),
                                   _ptr(vmax), _ptr(S), _ptr(ws), ws.numel(), _stream(stream))
    _check(rc, "wildcat_compress_kv")


def decode_workspace_bytes(shape) -> int:
    return int(lib().wc_decode_workspace_bytes(ctypes.byref(shape)))


def wildcat_decode(shape, opts, Q, KC, VC, WC, c_eff, vmin, vmax, O, ws, stream=None):
    units, _, C, d, tdt = _dims(shape)
    nq = shape.batch * shape.heads_q * shape.m * d
    dev = _need(KC, "KC", tdt, units * C * d)
    _need(VC, "VC", tdt, units * C * d, dev)
    _need(WC, "WC", torch.float32, units * C, dev)
    _need(c_eff, "c_eff", torch.int32, units, dev)
    _need(Q, "Q", tdt, nq, dev, exact=True, optional=nq == 0)
    _need(O, "O", tdt, nq, dev, exact=True, optional=nq == 0)
    _need(vmin, "vmin", tdt, units * d, dev)
    _need(vmax, "vmax", tdt, units * d, dev)
    _check_ws(ws, dev, decode_workspace_bytes(shape))
    rc = lib().wildcat_decode(ctypes.byref(shape), ctypes.byref(opts), _ptr(Q), _ptr(KC), _ptr(VC), _ptr(WC),
                              _ptr(c_eff), _ptr(vmin), _ptr(vmax), _ptr(O), _ptr(ws), 0 if ws is None else ws.numel(),
                              _stream(stream))
    _check(rc, "wildcat_decode")


def last_launch_count() -> int:
    return int(lib().wc_last_launch_count())


def timing_enable(on: bool = True) -> None:
    lib().wc_timing_enable(1 if on else 0)


def timing_read(cap: int = 8) -> list:
    buf = (ctypes.c_float * cap)()
    k = lib().wc_timing_read(buf, cap)
    if k < 0:
        raise WildcatError(f"wc_timing_read: {lib().wc_strerror(k).decode()}")
    return [float(buf[i]) for i in range(k)]


# ---------------------------------------------------------------- n-sharded path (PAR3)
def wc_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().wc_comm_unique_id(buf), "wc_comm_unique_id")
    return buf.raw


def wc_comm_init(uid: bytes, world: int, rank: int) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(uid, 128)
    _check(lib().wc_comm_init(ctypes.byref(h), buf, int(world), int(rank)), "wc_comm_init")
    return h


def wc_p2p_comm_create(world: int, rank: int, capacity: int):
    """Device-initiated (peer-memory) transport: returns (handle, this rank's 64-byte IPC handle)."""
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(64)
    _check(lib().wc_p2p_comm_create(ctypes.byref(h), int(world), int(rank), int(capacity), buf), "wc_p2p_comm_create")
    return h, buf.raw


def wc_p2p_comm_connect(h, handles: list) -> None:
    blob = ctypes.create_string_buffer(b"".join(handles), 64 * len(handles))
    _check(lib().wc_p2p_comm_connect(h, blob), "wc_p2p_comm_connect")


def wc_comm_destroy(h) -> None:
    _check(lib().wc_comm_destroy(h), "wc_comm_destroy")


def wildcat_forward_nshard(comm, shape, n_global, n_offset, opts, Q, K, V, O, S, r_eff, ws, stream=None):
    dev = _check_qkv(shape, Q, K, V, O, need_v=True, need_o=True)
    _need(S, "S", torch.int32, shape.r, dev, optional=True)
    _need(r_eff, "r_eff", torch.int32, 1, dev, optional=True)
    _check_ws(ws, dev, workspace_bytes(shape, WC_OP_FORWARD_NSHARD))
    rc = lib().wildcat_forward_nshard(comm, ctypes.byref(shape), int(n_global), int(n_offset), ctypes.byref(opts),
                                      _ptr(Q), _ptr(K), _ptr(V), _ptr(O), _ptr(S), _ptr(r_eff), _ptr(ws),
                                      ws.numel(), _stream(stream))
    _check(rc, "wildcat_forward_nshard")
