"""The C-ABI library without a GPU: it loads, exports every symbol that
include/maxmin.h declares, and rejects bad arguments before touching CUDA."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "maxmin.h")


@pytest.fixture(scope="module")
def L():
    from paper_cs_0610046_b200 import _build, _lib

    _build.build()
    return _lib.lib()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(maxmin_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert len(names) >= 10
    from paper_cs_0610046_b200 import _lib

    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (maxmin_\w+)", nm))
    for n in names:
        assert n in exported, n
        assert hasattr(L, n)
        assert n in _lib.SIGNATURES, f"binding lacks {n}"


def test_sass_is_sm100a():
    from paper_cs_0610046_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # TMA bulk copies global -> shared


def test_status_strings_and_sizes(L):
    assert L.maxmin_status_str(0) == b"ok"
    assert L.maxmin_status_str(7).startswith(b"output overlaps")
    assert [L.maxmin_dtype_size(d) for d in range(10)] == [1, 1, 2, 2, 4, 4, 8, 8, 4, 8]
    assert L.maxmin_dtype_size(10) == 0
    assert L.maxmin_version().startswith(b"maxmin-b200")


def test_workspace_query(L):
    b = ctypes.c_size_t(123)
    assert L.maxmin_workspace_bytes(8, 1, 1 << 28, 1024, ctypes.byref(b)) == 0 and b.value == 0
    assert L.maxmin_workspace_bytes(8, 1, 1 << 28, 65536, ctypes.byref(b)) == 0 and b.value > 0
    big = b.value
    assert L.maxmin_workspace_bytes(8, 4, 1 << 28, 65536, ctypes.byref(b)) == 0 and b.value > 3 * big
    assert L.maxmin_workspace_bytes(8, 1, 10, 0, ctypes.byref(b)) == 3
    assert L.maxmin_workspace_bytes(8, 1, 10, 11, ctypes.byref(b)) == 4
    assert L.maxmin_workspace_bytes(12, 1, 10, 3, ctypes.byref(b)) == 2
    hb = ctypes.c_size_t(0)
    assert L.maxmin_host_workspace_bytes(8, 1 << 28, 1024, 0, ctypes.byref(hb)) == 0 and hb.value > 0


P = 0x7F0000000000  # fake, 16-B aligned device-like addresses: validation runs before CUDA


def call_1d(L, dt=8, inp=P, n=1000, w=10, omax=P + (1 << 20), omin=P + (2 << 20), ws=None, wsb=0):
    return L.maxmin_filter_1d(dt, inp, n, w, omax, omin, ws, wsb, None)


def test_argument_errors_before_cuda(L):
    assert call_1d(L, dt=11) == 2                       # dtype
    assert call_1d(L, inp=None) == 1                    # null input
    assert call_1d(L, omax=None, omin=None) == 1        # both outputs null
    assert call_1d(L, w=0) == 3                         # w < 1
    assert call_1d(L, w=1001) == 4                      # w > n
    assert call_1d(L, n=0, w=1) == 5                    # n < 1
    assert call_1d(L, inp=P + 4) == 6                   # misaligned input
    assert call_1d(L, omax=P + (1 << 20) + 8) == 6      # misaligned output
    assert call_1d(L, omax=P + 400) == 7                # output overlaps input
    assert call_1d(L, omax=P + (1 << 20), omin=P + (1 << 20) + 16) == 7  # outputs overlap
    assert call_1d(L, n=1 << 20, w=100000, omax=P + (16 << 20), omin=P + (32 << 20)) == 8  # needs workspace
    # batched: ld checks and per-row alignment
    assert L.maxmin_filter_batched(8, P, 4, 100, 99, 10, P + (1 << 20), None, 91, None, 0, None) == 5
    assert L.maxmin_filter_batched(8, P, 4, 100, 100, 10, P + (1 << 20), None, 90, None, 0, None) == 5
    assert L.maxmin_filter_batched(8, P, 4, 100, 101, 10, P + (1 << 20), None, 92, None, 0, None) == 6
    assert L.maxmin_filter_batched(8, P, 0, 100, 100, 10, P + (1 << 20), None, 92, None, 0, None) == 0
    # 2-D
    f2 = L.maxmin_filter_2d
    assert f2(0, P, 1, 10, 10, 16, 160, 3, 11, P + (1 << 20), None, 16, 160, None) == 4
    assert f2(0, P, 1, 10, 10, 16, 160, 0, 3, P + (1 << 20), None, 16, 160, None) == 3
    assert f2(8, P + 2, 1, 10, 10, 12, 120, 3, 3, P + (1 << 20), None, 16, 160, None) == 6
    assert f2(0, P, 1, 10, 10, 12, 120, 3, 3, P + (1 << 20), None, 16, 160, None) != 6  # u8: any ld
    assert f2(0, P, 2, 10, 10, 16, 100, 3, 3, P + (1 << 20), None, 16, 160, None) == 5
    assert f2(0, P, 1, 10, 10, 16, 160, 3, 3, P + 32, None, 16, 160, None) == 7
    assert f2(0, P, 0, 10, 10, 16, 160, 3, 3, P + (1 << 20), None, 16, 160, None) == 0


def test_binding_raises_without_fallback():
    import paper_cs_0610046_b200 as mm
    import torch

    with pytest.raises((ValueError, mm.MaxMinError, RuntimeError)):
        mm.maxmin_filter_1d(torch.zeros(100), 3)  # CPU tensor: no CPU path exists


def test_argfilter_argument_errors(L):
    """N1 entry points: every argument error is reported before any launch."""
    b = ctypes.c_size_t(0)
    assert L.maxmin_argfilter_workspace_bytes(8, 1, 1000, 10, ctypes.byref(b)) == 0 and b.value == 0  # fused
    assert L.maxmin_argfilter_workspace_bytes(8, 1, 5000, 2000, ctypes.byref(b)) == 0 and b.value > 32 * 3000
    assert L.maxmin_argfilter_workspace_bytes(9, 1, 1000, 10, ctypes.byref(b)) == 10  # f64: unsupported
    assert L.maxmin_argfilter_workspace_bytes(8, 1, 10, 0, ctypes.byref(b)) == 3
    assert L.maxmin_argfilter_workspace_bytes(8, 1, 10, 11, ctypes.byref(b)) == 4
    assert L.maxmin_argfilter_workspace_bytes(12, 1, 10, 3, ctypes.byref(b)) == 2
    f = L.maxmin_argfilter_batched
    P = 1 << 30  # fake addresses: every error below is found before any access
    assert f(8, None, 1, 100, 100, 10, P + (1 << 24), None, None, None, 91, P + (1 << 26), 1 << 20, None) == 1
    assert f(8, P, 1, 100, 100, 10, None, None, None, None, 91, P + (1 << 26), 1 << 20, None) == 1
    assert f(8, P, 1, 100, 100, 10, None, None, P + (1 << 24) + 4, None, 91, P + (1 << 26), 1 << 20, None) == 6
    assert f(8, P, 1, 5000, 5000, 2000, None, None, P + (1 << 24), None, 3001, None, 0, None) == 8
    assert f(8, P, 1, 100, 100, 10, None, None, P + 8, None, 91, P + (1 << 26), 1 << 20, None) == 7
    assert f(9, P, 1, 100, 100, 10, None, None, P + (1 << 24), None, 91, P + (1 << 26), 1 << 20, None) == 10


def test_stream_argument_errors(L):
    """N2 entry points: argument errors are reported before any CUDA call."""
    from paper_cs_0610046_b200 import _lib

    b = ctypes.c_size_t(0)
    assert L.maxmin_stream_state_bytes(8, 65536, 129, 256, ctypes.byref(b)) == 0
    assert b.value >= 2 * 65536 * 128 * 4  # fused path: two history rows of w-1 samples
    assert L.maxmin_stream_state_bytes(12, 4, 3, 8, ctypes.byref(b)) == 2
    assert L.maxmin_stream_state_bytes(8, 4, 0, 8, ctypes.byref(b)) == 3
    assert L.maxmin_stream_state_bytes(8, 4, 3, 0, ctypes.byref(b)) == 5
    assert L.maxmin_stream_state_bytes(8, -1, 3, 8, ctypes.byref(b)) == 5
    st = _lib.Stream()
    P = 1 << 30
    L.maxmin_stream_state_bytes(8, 4, 3, 8, ctypes.byref(b))
    assert L.maxmin_stream_init(None, 8, 4, 3, 8, P, b.value, None) == 1
    assert L.maxmin_stream_init(ctypes.byref(st), 8, 4, 3, 8, None, b.value, None) == 1
    assert L.maxmin_stream_init(ctypes.byref(st), 8, 4, 3, 8, P + 4, b.value, None) == 6
    assert L.maxmin_stream_init(ctypes.byref(st), 8, 4, 3, 8, P, b.value - 1, None) == 8
    # a zero-stream state needs no device memory: init and push are no-ops
    assert L.maxmin_stream_init(ctypes.byref(st), 8, 0, 3, 8, None, 0, None) == 0
    fv = ctypes.c_int64(-1)
    assert L.maxmin_stream_push(ctypes.byref(st), None, 5, 0, None, None, 8, ctypes.byref(fv), None) == 0
    assert fv.value == 2 and st.seen == 0  # w-1 = 2 samples short; nothing ingested with no streams
    assert L.maxmin_stream_push(ctypes.byref(st), None, 9, 0, None, None, 8, ctypes.byref(fv), None) == 5
    assert L.maxmin_stream_push(ctypes.byref(st), None, -1, 0, None, None, 8, ctypes.byref(fv), None) == 5
    assert L.maxmin_stream_push(ctypes.byref(st), None, 1, 0, None, None, 8, None, None) == 1


def test_3d_argument_errors(L):
    b = ctypes.c_size_t(0)
    assert L.maxmin_filter_3d_workspace_bytes(8, 10, 20, 30, 32, 3, 3, 3, ctypes.byref(b)) == 0 and b.value >= 2 * 8 * 640 * 4
    assert L.maxmin_filter_3d_workspace_bytes(8, 10, 20, 30, 29, 3, 3, 3, ctypes.byref(b)) == 5  # in_ld < cols
    assert L.maxmin_filter_3d_workspace_bytes(8, 10, 20, 30, 32, 3, 3, 11, ctypes.byref(b)) == 4
    f = L.maxmin_filter_3d
    P = 1 << 30
    assert f(8, None, 10, 20, 30, 32, 640, 3, 3, 3, P + (1 << 24), None, 28, 560, P + (1 << 26), 1 << 20, None) == 1
    assert f(8, P, 10, 20, 30, 32, 640, 0, 3, 3, P + (1 << 24), None, 28, 560, P + (1 << 26), 1 << 20, None) == 3
    assert f(8, P, 10, 20, 30, 32, 640, 31, 3, 3, P + (1 << 24), None, 28, 560, P + (1 << 26), 1 << 20, None) == 4
    assert f(8, P, 10, 20, 30, 32, 600, 3, 3, 3, P + (1 << 24), None, 28, 560, P + (1 << 26), 1 << 20, None) == 5
    assert f(8, P, 10, 20, 30, 32, 640, 3, 3, 3, P + (1 << 24) + 2, None, 28, 560, P + (1 << 26), 1 << 20, None) == 6
    assert f(8, P, 10, 20, 30, 32, 640, 3, 3, 3, P + (1 << 24), None, 28, 560, None, 0, None) == 8
    assert f(8, P, 10, 20, 30, 32, 640, 3, 3, 3, P + 64, None, 28, 560, P + (1 << 26), 1 << 20, None) == 7


def test_2d_ws_argument_errors(L):
    b = ctypes.c_size_t(0)
    assert L.maxmin_filter_2d_workspace_bytes(8, 2, 100, 120, 5, 7, ctypes.byref(b)) == 0 and b.value >= 2 * 2 * 100 * 116 * 4
    assert L.maxmin_filter_2d_workspace_bytes(0, 2, 100, 120, 15, 15, ctypes.byref(b)) == 0 and b.value == 0  # packed bytes
    assert L.maxmin_filter_2d_workspace_bytes(8, 2, 100, 120, 5, 17, ctypes.byref(b)) == 0 and b.value == 0  # w_col > 16
    assert L.maxmin_filter_2d_workspace_bytes(8, 2, 100, 120, 0, 7, ctypes.byref(b)) == 3
    assert L.maxmin_filter_2d_workspace_bytes(8, 2, 100, 120, 121, 7, ctypes.byref(b)) == 4
    f = L.maxmin_filter_2d_ws
    P = 1 << 30
    assert f(8, None, 1, 10, 10, 16, 160, 3, 3, P + (1 << 20), None, 16, 160, None, 0, None) == 1
    assert f(8, P, 1, 10, 10, 16, 160, 3, 3, P + (1 << 20), None, 16, 160, P + (1 << 24) + 4, 1 << 20, None) == 8
    assert f(8, P, 1, 10, 10, 16, 160, 3, 3, P + 32, None, 16, 160, None, 0, None) == 7
