"""C ABI checks that need no GPU: the library builds and loads, exports every symbol declared in
include/wildcat.h, and rejects invalid arguments before any CUDA call (nothing is launched)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "wildcat.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\**\s*(\w+)\s*\(", src, flags=re.M)) - {"if"})


@pytest.fixture(scope="module")
def L():
    import paper_2602_10056_b200 as wc

    return wc.lib()


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert {"wildcat_select", "wildcat_weights", "wildcat_attend", "wildcat_forward"} <= set(names)
    for nm in names:
        assert hasattr(L, nm), nm


def test_library_is_sm100a():
    import paper_2602_10056_b200.build as b

    assert "arch=compute_100a,code=sm_100a" in " ".join(b.NVCC_FLAGS)
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {b.LIB} 2>/dev/null").read()
    assert "sm_100a" in out


def _shape(**kw):
    from paper_2602_10056_b200 import _binding as B

    base = dict(batch=1, heads_q=1, heads_kv=1, d=64, r=8, bins=1, dtype=1, reserved=0, m=16, n=100)
    base.update(kw)
    return B.wc_shape(**base)


@pytest.mark.parametrize("kw,code", [
    (dict(r=0), -2), (dict(r=101), -2), (dict(d=48), -2), (dict(heads_q=3, heads_kv=2), -2),
    (dict(dtype=7), -3), (dict(bins=9), -2), (dict(bins=0), -2), (dict(m=-1), -2),
    (dict(n=0), -2),
])
def test_validation_before_launch(L, kw, code):
    from paper_2602_10056_b200 import _binding as B

    s = _shape(**kw)
    o = B.make_opts()
    dummy = ctypes.c_void_p(0x1000)
    rc = L.wildcat_forward(ctypes.byref(s), ctypes.byref(o), dummy, dummy, dummy, dummy, None, None, dummy, 1 << 30,
                           None)
    assert rc == code
    assert L.wc_workspace_bytes(ctypes.byref(s), 3) == 0


def test_null_and_workspace_errors(L):
    from paper_2602_10056_b200 import _binding as B

    s = _shape()
    o = B.make_opts()
    d = ctypes.c_void_p(0x1000)
    assert L.wildcat_forward(ctypes.byref(s), ctypes.byref(o), d, None, d, d, None, None, d, 1 << 30, None) == -1
    need = L.wc_workspace_bytes(ctypes.byref(s), 3)
    assert need > 0
    assert L.wildcat_forward(ctypes.byref(s), ctypes.byref(o), d, d, d, d, None, None, d, need - 1, None) == -4
    assert L.wildcat_forward(ctypes.byref(s), ctypes.byref(o), d, d, d, d, None, None,
                             ctypes.c_void_p(0x1001), 1 << 40, None) == -4
    # rq < 0 requires Q
    assert L.wildcat_select(ctypes.byref(s), ctypes.byref(o), None, d, d, d, d, d, d, 1 << 40, None) == -1
    assert L.wc_strerror(-2).decode().startswith("invalid shape")


def test_workspace_sizes_scale(L):
    s1 = _shape(n=1000, r=10)
    s2 = _shape(n=2000, r=20)
    # n x r grows 4x; the blocked selection's F rows come in quads (r rounded up to a multiple of 4),
    # which weighs more at r = 10 than at r = 20, and the per-unit scalars do not grow
    assert L.wc_workspace_bytes(ctypes.byref(s2), 0) > 2.5 * L.wc_workspace_bytes(ctypes.byref(s1), 0)
    big_m = _shape(n=1000, r=10, m=500)
    assert L.wc_workspace_bytes(ctypes.byref(big_m), 2) > 0  # tcgen05 attend: per-unit operand image
    assert L.wc_workspace_bytes(ctypes.byref(_shape(n=1000, r=10, m=500, dtype=0)), 2) == 0  # fp32: none
    assert L.wc_workspace_bytes(ctypes.byref(_shape(n=1000, r=10, m=16)), 2) > 0  # decode kernel partials


def test_kv_cache_abi(L):
    from paper_2602_10056_b200 import _binding as B

    # capacity C = keep_first + keep_last + B * min(ceil(r/B), n_mid/B) (reading Z24)
    s = _shape(n=1000, r=64)
    assert B.kv_capacity(s, 32, 32) == 64 + 64
    assert B.kv_capacity(s, 500, 500) == 1000  # nothing compressed
    assert B.kv_capacity(_shape(n=1000, r=64, bins=4), 20, 20) == 40 + 64
    # 5 bins do not divide n_mid = 936: bins of 187 keys (the last 188), rb = 13 (Z13)
    assert B.kv_capacity(_shape(n=1000, r=64, bins=5), 32, 32) == 64 + 5 * 13
    assert B.kv_capacity(s, 600, 500) == 0 and B.kv_capacity(s, -1, 0) == 0
    assert B.kv_workspace_bytes(s, 32, 32) > 0
    o = B.make_opts()
    d = ctypes.c_void_p(0x1000)
    f = ctypes.c_void_p(0x1000)
    # invalid split -> WC_ESHAPE; null cache output -> WC_EINVAL; small workspace -> WC_EWORKSPACE
    assert L.wildcat_compress_kv(ctypes.byref(s), ctypes.byref(o), 600, 500, d, d, d, d, d, f, d, d, d, None, d,
                                 1 << 40, None) == -2
    assert L.wildcat_compress_kv(ctypes.byref(s), ctypes.byref(o), 32, 32, d, d, d, None, d, f, d, d, d, None, d,
                                 1 << 40, None) == -1
    need = B.kv_workspace_bytes(s, 32, 32)
    assert L.wildcat_compress_kv(ctypes.byref(s), ctypes.byref(o), 32, 32, d, d, d, d, d, f, d, d, d, None, d,
                                 need - 1, None) == -4
    # more bins than the middle has keys (n_mid = 36 < 40 bins, r = 64): rejected before any launch
    assert L.wildcat_compress_kv(ctypes.byref(_shape(n=100, r=64, bins=40)), ctypes.byref(o), 32, 32, d, d, d, d, d, f,
                                 d, d, d, None, d, 1 << 40, None) == -2


def test_product_package_has_no_oracle_dependency():
    # the product path must never import or link the oracle (test infrastructure only)
    pkg = os.path.join(ROOT, "paper_2602_10056_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "wildcat_oracle" not in txt, fn


def test_block_option_validation(L):
    from paper_2602_10056_b200 import _binding as B

    assert ctypes.sizeof(B.wc_opts) == 40
    d = ctypes.c_void_p(0x1000)
    s = _shape()
    o = B.make_opts(block=33)  # > WC_MAX_BLOCK
    assert L.wildcat_forward(ctypes.byref(s), ctypes.byref(o), d, d, d, d, None, None, d, 1 << 40, None) == -1
    assert L.wc_version() >= 101


@pytest.mark.parametrize("block", [1, 8])
def test_r_above_max_r_is_unsupported_on_every_path(L, block):
    # WC_MAX_R = 1024: the r x r solve and the blocked plan are sized for it; larger r (or rb per bin)
    # must be refused before any launch on every selection path, sequential included
    from paper_2602_10056_b200 import _binding as B

    d = ctypes.c_void_p(0x1000)
    o = B.make_opts(block=block)
    for r in (1025, 2048):
        big = _shape(n=5000, r=r)
        assert L.wildcat_forward(ctypes.byref(big), ctypes.byref(o), d, d, d, d, None, None, d, 1 << 40, None) == -7
        assert L.wildcat_select(ctypes.byref(big), ctypes.byref(o), d, d, d, d, d, d, d, 1 << 40, None) == -7
        assert L.wildcat_weights(ctypes.byref(big), ctypes.byref(o), d, d, d, d, d, d, d, d, d, d, d, 1 << 40,
                                 None) == -7
        assert L.wildcat_compress_kv(ctypes.byref(big), ctypes.byref(o), 32, 32, d, d, d, d, d, d, d, d, d, None, d,
                                     1 << 40, None) == -7
        assert L.wildcat_forward_nshard(d, ctypes.byref(big), 5000, 0, ctypes.byref(o), d, d, d, d, None, None, d,
                                        1 << 40, None) == -7
    # with bins, the limit applies per bin: r = 2048 over 2 bins is rb = 1024 (accepted by the check)
    ok = _shape(n=5000, r=2048, bins=2)
    assert L.wc_workspace_bytes(ctypes.byref(ok), 3) > 0


def test_binding_refuses_cpu_tensors():
    # the ctypes wrappers refuse tensors that are not CUDA before any C call (no CPU fallback);
    # the shape / dtype / size rules are exercised on the GPU in tests/test_gpu_parity.py
    import torch

    from paper_2602_10056_b200 import _binding as B

    s = _shape(n=100, r=8, m=16)
    K = torch.zeros(1, 1, 100, 64, dtype=torch.bfloat16)
    with pytest.raises(B.WildcatError, match="CUDA"):
        B._check_qkv(s, K, K)
    with pytest.raises(B.WildcatError, match="torch.Tensor"):
        B._need(object(), "X", torch.float32, 1)
    with pytest.raises(B.WildcatError, match="required"):
        B._need(None, "X", torch.float32, 1)


def test_unknown_flag_and_version(L):
    from paper_2602_10056_b200 import _binding as B

    s = _shape()
    o = B.make_opts()
    o.flags = 1 << 7  # not a WC_* flag
    d = ctypes.c_void_p(0x1000)
    need = L.wc_workspace_bytes(ctypes.byref(s), 3)
    assert L.wildcat_forward(ctypes.byref(s), ctypes.byref(o), d, d, d, d, None, None, d, need, None) == -1
    assert L.wc_version() == 201
    assert ctypes.sizeof(B.wc_opts) == 40  # beta, rq, seed, flags, block, unit_offset
    assert L.wc_strerror(-8).decode().startswith("non-finite")


def test_block32_plan_limit(L):
    """16 < b <= 32 runs the 32-slot plan, whose candidate columns must fit shared memory: r = 1024
    is refused before any launch (WC_EUNSUPPORTED), r = 256 accepted by validation."""
    from paper_2602_10056_b200 import _binding as B

    d = ctypes.c_void_p(0x1000)
    big = _shape(n=5000, r=1024, d=128)
    o = B.make_opts(block=32)
    assert L.wildcat_forward(ctypes.byref(big), ctypes.byref(o), d, d, d, d, None, None, d, 1 << 40, None) == -7
    o16 = B.make_opts(block=16)
    small = _shape(n=5000, r=256, d=128)
    need = L.wc_workspace_bytes(ctypes.byref(small), 3)
    # r = 256 passes every check; with a too-small workspace the call stops at the workspace check
    assert L.wildcat_forward(ctypes.byref(small), ctypes.byref(o), d, d, d, d, None, None, d, need - 1, None) == -4
    assert L.wildcat_forward(ctypes.byref(big), ctypes.byref(o16), d, d, d, d, None, None, d, 1 << 10, None) == -4
