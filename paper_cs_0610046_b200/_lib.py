"""ctypes loader for libmaxmin.so (the C ABI declared in include/maxmin.h).

There is no fallback: if the CUDA library is missing or fails to load, every
call raises.  Argument marshalling only -- all filtering runs in the library.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MAXMIN_LIB selects another in-tree build (A/B experiments); default libmaxmin.so
LIB_PATH = os.path.join(_HERE, os.environ.get("MAXMIN_LIB", "libmaxmin.so"))

# maxmin_dtype (include/maxmin.h)
U8, I8, U16, I16, U32, I32, U64, I64, F32, F64 = range(10)

STATUS = {
    0: "ok", 1: "null pointer", 2: "unknown dtype", 3: "window < 1",
    4: "window larger than input", 5: "bad shape", 6: "misaligned pointer or leading dimension",
    7: "output overlaps input or the other output", 8: "workspace missing or too small",
    9: "CUDA error", 10: "unsupported by this build", 11: "pointer is not device memory",
    12: "data pointers on different devices", 13: "NCCL error",
}


class MaxMinError(RuntimeError):
    def __init__(self, status: int, cuda_error: int = 0, nccl_error: int = 0):
        msg = f"maxmin status {status}: {STATUS.get(status, 'unknown')}"
        if status == 9:
            msg += f" (cudaError {cuda_error})"
        if status == 13:
            msg += f" (ncclResult {nccl_error})"
        super().__init__(msg)
        self.status = status
        self.cuda_error = cuda_error
        self.nccl_error = nccl_error


_lib = None
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t


class Stream(ctypes.Structure):
    """maxmin_stream (include/maxmin.h): host-side description of N2 stream state."""
    _fields_ = [("dtype", ctypes.c_int32), ("phase", ctypes.c_int32), ("streams", _i64), ("w", _i64),
                ("max_chunk", _i64), ("ld", _i64), ("seen", _i64), ("state", _vp), ("state_bytes", _sz)]


_sp = ctypes.POINTER(Stream)

SIGNATURES = {
    "maxmin_status_str": (ctypes.c_char_p, [ctypes.c_int]),
    "maxmin_last_cuda_error": (ctypes.c_int, []),
    "maxmin_version": (ctypes.c_char_p, []),
    "maxmin_dtype_size": (_sz, [ctypes.c_int]),
    "maxmin_workspace_bytes": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i64, ctypes.POINTER(_sz)]),
    "maxmin_filter_1d": (ctypes.c_int, [ctypes.c_int, _vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "maxmin_filter_batched": (ctypes.c_int, [ctypes.c_int, _vp, _i64, _i64, _i64, _i64, _vp, _vp,
                                             _i64, _vp, _sz, _vp]),
    "maxmin_filter_2d": (ctypes.c_int, [ctypes.c_int, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _i64,
                                        _vp, _vp, _i64, _i64, _vp]),
    "maxmin_argfilter_workspace_bytes": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i64, ctypes.POINTER(_sz)]),
    "maxmin_argfilter_batched": (ctypes.c_int, [ctypes.c_int, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp,
                                                _vp, _i64, _vp, _sz, _vp]),
    "maxmin_lb_keogh_batched": (ctypes.c_int, [ctypes.c_int, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _vp]),
    "maxmin_stream_state_bytes": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i64, ctypes.POINTER(_sz)]),
    "maxmin_stream_init": (ctypes.c_int, [_sp, ctypes.c_int, _i64, _i64, _i64, _vp, _sz, _vp]),
    "maxmin_stream_push": (ctypes.c_int, [_sp, _vp, _i64, _i64, _vp, _vp, _i64, ctypes.POINTER(_i64), _vp]),
    "maxmin_morph_batched": (ctypes.c_int, [ctypes.c_int, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _vp]),
    "maxmin_morph_2d_workspace_bytes": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i64, _i64, _i64,
                                                       ctypes.POINTER(_sz)]),
    "maxmin_morph_2d": (ctypes.c_int, [ctypes.c_int, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _vp,
                                       _i64, _i64, _vp, _sz, _vp]),
    "maxmin_filter_3d_workspace_bytes": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i64, _i64, _i64, _i64, _i64,
                                                        ctypes.POINTER(_sz)]),
    "maxmin_filter_2d_workspace_bytes": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i64, _i64, _i64,
                                                        ctypes.POINTER(_sz)]),
    "maxmin_filter_2d_ws": (ctypes.c_int, [ctypes.c_int, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _i64,
                                           _vp, _vp, _i64, _i64, _vp, _sz, _vp]),
    "maxmin_filter_3d": (ctypes.c_int, [ctypes.c_int, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _vp,
                                        _i64, _i64, _vp, _sz, _vp]),
    "maxmin_host_workspace_bytes": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i64, ctypes.POINTER(_sz)]),
    "maxmin_filter_1d_host": (ctypes.c_int, [ctypes.c_int, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _sz]),
    "maxmin_sharded_workspace_bytes": (ctypes.c_int, [ctypes.c_int, _i64, _i64, ctypes.POINTER(_i64), ctypes.c_int,
                                                      ctypes.POINTER(_sz)]),
    "maxmin_filter_1d_sharded": (ctypes.c_int, [ctypes.c_int, _vp, _i64, _i64, ctypes.POINTER(_i64), ctypes.c_int,
                                                ctypes.c_int, ctypes.c_int, _vp, ctypes.POINTER(_vp),
                                                ctypes.POINTER(_vp), _vp, _sz, _vp, _vp]),
    "maxmin_last_nccl_error": (ctypes.c_int, []),
}


def lib():
    """Load libmaxmin.so (raises if it is missing: no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() "
                              "(python paper_cs_0610046_b200/_build.py)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        L = lib()
        raise MaxMinError(status, L.maxmin_last_cuda_error(), L.maxmin_last_nccl_error() if status == 13 else 0)
