"""B200-native running max-min filter (arXiv cs/0610046).

Python binding of libmaxmin.so with the names of the C ABI (include/maxmin.h).
Marshalling only: tensors are PyTorch CUDA tensors (device memory + the current
stream); every step of the filter runs in the library's sm_100a kernels.  There
is no CPU fallback -- a missing library raises.

    out_max[j] = max a[j .. j+w)   out_min[j] = min a[j .. j+w)
"""
from __future__ import annotations

import ctypes
import functools

import torch

from . import _lib
from ._lib import MaxMinError

__all__ = [
    "MaxMinError", "dtype_code", "maxmin_workspace_bytes", "maxmin_filter_1d",
    "maxmin_filter_batched", "maxmin_filter_2d", "maxmin_filter_1d_host",
    "maxmin_host_workspace_bytes", "maxmin_argfilter_workspace_bytes", "maxmin_argfilter_batched",
    "maxmin_argfilter_1d", "maxmin_lb_keogh_batched", "maxmin_stream_state_bytes", "MaxMinStream", "maxmin_morph_batched",
    "maxmin_morph_1d", "maxmin_morph_2d", "maxmin_filter_3d", "maxmin_sharded_workspace_bytes",
    "maxmin_filter_1d_sharded", "version",
]

_CODES = {
    torch.uint8: _lib.U8, torch.int8: _lib.I8, torch.uint16: _lib.U16, torch.int16: _lib.I16,
    torch.uint32: _lib.U32, torch.int32: _lib.I32, torch.uint64: _lib.U64, torch.int64: _lib.I64,
    torch.float32: _lib.F32, torch.float64: _lib.F64,
}


def dtype_code(dtype) -> int:
    try:
        return _CODES[dtype]
    except KeyError:
        raise TypeError(f"maxmin: unsupported dtype {dtype}") from None


def version() -> str:
    return _lib.lib().maxmin_version().decode()


try:  # the raw handle of the current stream without building a Stream object (~0.3 us)
    _raw_stream = torch._C._cuda_getCurrentRawStream
except AttributeError:  # pragma: no cover
    _raw_stream = None


def _stream_ptr(stream, device=None) -> ctypes.c_void_p:
    if stream is None:
        if _raw_stream is not None:
            idx = torch.cuda.current_device() if device is None or device.index is None else device.index
            return ctypes.c_void_p(_raw_stream(idx))
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _check_out(name: str, t, x: torch.Tensor, shape) -> None:
    """A caller-supplied output: the input's dtype and device, at least `shape`
    (leading dims exact, last dim >= shape[-1]) and unit stride along the last
    dim -- the C ABI cannot see buffer sizes, so an undersized or mistyped output
    would be written past its end."""
    if t is None:
        return
    if t.dtype != x.dtype or t.device != x.device:
        raise ValueError(f"{name}: dtype/device {t.dtype}/{t.device} differ from the input's {x.dtype}/{x.device}")
    if t.dim() != len(shape) or tuple(t.shape[:-1]) != tuple(shape[:-1]) or t.shape[-1] < shape[-1]:
        raise ValueError(f"{name}: shape {tuple(t.shape)} does not hold {tuple(shape)}")
    if shape[-1] > 0 and t.stride(-1) != 1:
        raise ValueError(f"{name}: the last dimension must be contiguous")


def _pair_strides(name: str, a, b, dims: int) -> None:
    """Both outputs share one row (and image) stride: the C ABI takes one pitch."""
    if a is not None and b is not None and tuple(a.stride()[:dims]) != tuple(b.stride()[:dims]):
        raise ValueError(f"{name}: out_max and out_min must have the same strides")


def _alloc_out(ref, shape, dtype, device):
    """A fresh output of `shape`: with the strides of `ref` (the caller's other
    output) when given, so both share one pitch; else rows padded to 16 bytes."""
    if ref is not None:
        return torch.empty_strided(tuple(shape), tuple(ref.stride()), dtype=dtype, device=device)
    vec = max(16 // torch.empty((), dtype=dtype).element_size(), 1)
    pad = (shape[-1] + vec - 1) // vec * vec
    return torch.empty(*shape[:-1], pad, dtype=dtype, device=device)[..., : shape[-1]]


@functools.lru_cache(maxsize=256)
def _workspace_bytes(code: int, batch: int, n: int, w: int) -> int:
    out = ctypes.c_size_t(0)
    _lib.check(_lib.lib().maxmin_workspace_bytes(code, batch, n, w, ctypes.byref(out)))
    return int(out.value)


def maxmin_workspace_bytes(dtype, batch: int, n: int, w: int) -> int:
    return _workspace_bytes(dtype_code(dtype), batch, n, w)


def _workspace(dtype, batch, n, w, device, workspace):
    need = maxmin_workspace_bytes(dtype, batch, n, w)
    if need == 0:
        return None, 0
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=device)
    return workspace, workspace.numel() * workspace.element_size()


def maxmin_filter_1d(x: torch.Tensor, w: int, out_max=None, out_min=None, *, want_max=True,
                     want_min=True, workspace=None, stream=None):
    """Running max and min of a contiguous 1-D CUDA tensor; returns (out_max, out_min)."""
    if x.dim() != 1 or not x.is_cuda or not x.is_contiguous():
        raise ValueError("maxmin_filter_1d: x must be a contiguous 1-D CUDA tensor")
    n = x.shape[0]
    m = max(n - w + 1, 0)
    _check_out("out_max", out_max, x, (m,))
    _check_out("out_min", out_min, x, (m,))
    if want_max and out_max is None and m > 0:
        out_max = torch.empty(m, dtype=x.dtype, device=x.device)
    if want_min and out_min is None and m > 0:
        out_min = torch.empty(m, dtype=x.dtype, device=x.device)
    ws, wsb = _workspace(x.dtype, 1, n, w, x.device, workspace) if 1 <= w <= n else (None, 0)
    _lib.check(_lib.lib().maxmin_filter_1d(dtype_code(x.dtype), _ptr(x), n, w, _ptr(out_max),
                                           _ptr(out_min), _ptr(ws), wsb, _stream_ptr(stream, x.device)))
    return out_max, out_min


def maxmin_filter_batched(x: torch.Tensor, w: int, n: int | None = None, out_max=None, out_min=None,
                          *, want_max=True, want_min=True, workspace=None, stream=None):
    """The 1-D filter on every row of a 2-D CUDA tensor [batch, ld] (first n columns)."""
    if x.dim() != 2 or not x.is_cuda or x.stride(1) != 1:
        raise ValueError("maxmin_filter_batched: x must be a row-major 2-D CUDA tensor")
    batch, ncols = x.shape
    n = ncols if n is None else n
    m = max(n - w + 1, 0)
    _check_out("out_max", out_max, x, (batch, m))
    _check_out("out_min", out_min, x, (batch, m))
    _pair_strides("maxmin_filter_batched", out_max, out_min, 1)
    # rows of fresh outputs are padded to 16 bytes (the C ABI's alignment rule),
    # or take the pitch of the output the caller supplied
    if want_max and out_max is None and m > 0:
        out_max = _alloc_out(out_min, (batch, m), x.dtype, x.device)
    if want_min and out_min is None and m > 0:
        out_min = _alloc_out(out_max, (batch, m), x.dtype, x.device)
    out_ld = (out_max if out_max is not None else out_min).stride(0) if m > 0 else 1
    ws, wsb = _workspace(x.dtype, batch, n, w, x.device, workspace) if 1 <= w <= n else (None, 0)
    _lib.check(_lib.lib().maxmin_filter_batched(dtype_code(x.dtype), _ptr(x), batch, n, x.stride(0), w,
                                                _ptr(out_max), _ptr(out_min), out_ld, _ptr(ws), wsb,
                                                _stream_ptr(stream, x.device)))
    return out_max, out_min


@functools.lru_cache(maxsize=256)
def _workspace_2d(code: int, batch: int, rows: int, cols: int, w_row: int, w_col: int) -> int:
    out = ctypes.c_size_t(0)
    _lib.check(_lib.lib().maxmin_filter_2d_workspace_bytes(code, batch, rows, cols, w_row, w_col, ctypes.byref(out)))
    return int(out.value)


def maxmin_filter_2d(x: torch.Tensor, w_row: int, w_col: int, cols: int | None = None, out_max=None,
                     out_min=None, *, want_max=True, want_min=True, workspace=None, stream=None):
    """Separable 2-D max/min over a [batch, rows, ld] (or [rows, ld]) CUDA tensor.

    Output (b, r, c) covers rows [r, r+w_col) x columns [c, c+w_row); only the valid
    region (rows-w_col+1) x (cols-w_row+1) is computed.  Outside the packed-byte
    kernel's domain (1-byte pixels, square windows <= 17) the separable path needs
    scratch of two row-filtered images (maxmin_filter_2d_workspace_bytes); pass
    `workspace` to reuse a buffer, else one is allocated from torch's caching allocator.
    """
    squeeze = x.dim() == 2
    xx = x[None] if squeeze else x
    if xx.dim() != 3 or not xx.is_cuda or xx.stride(2) != 1:
        raise ValueError("maxmin_filter_2d: x must be a row-major [batch, rows, ld] CUDA tensor")
    batch, rows, ld = xx.shape
    cols = ld if cols is None else cols
    R, C = rows - w_col + 1, cols - w_row + 1
    if squeeze:  # [rows, ld] input: outputs may be given as [R, C]
        out_max = out_max[None] if out_max is not None and out_max.dim() == 2 else out_max
        out_min = out_min[None] if out_min is not None and out_min.dim() == 2 else out_min
    _check_out("out_max", out_max, x, (batch, max(R, 0), max(C, 0)))
    _check_out("out_min", out_min, x, (batch, max(R, 0), max(C, 0)))
    _pair_strides("maxmin_filter_2d", out_max, out_min, 2)
    if want_max and out_max is None and R > 0 and C > 0:
        out_max = _alloc_out(out_min, (batch, R, C), x.dtype, x.device)
    if want_min and out_min is None and R > 0 and C > 0:
        out_min = _alloc_out(out_max, (batch, R, C), x.dtype, x.device)
    om = out_max if out_max is not None else out_min
    out_ld = om.stride(1) if om is not None else 1
    out_bs = om.stride(0) if om is not None else 1
    need = _workspace_2d(dtype_code(x.dtype), batch, rows, cols, w_row, w_col) if R > 0 and C > 0 else 0
    if workspace is None and need:
        workspace = torch.empty(need, dtype=torch.uint8, device=x.device)
    _lib.check(_lib.lib().maxmin_filter_2d_ws(dtype_code(x.dtype), _ptr(xx), batch, rows, cols,
                                              xx.stride(1), xx.stride(0), w_row, w_col, _ptr(out_max),
                                              _ptr(out_min), out_ld, out_bs, _ptr(workspace),
                                              0 if workspace is None else workspace.numel(),
                                              _stream_ptr(stream, x.device)))
    if squeeze:
        out_max = out_max[0] if out_max is not None and out_max.dim() == 3 else out_max
        out_min = out_min[0] if out_min is not None and out_min.dim() == 3 else out_min
    return out_max, out_min


def maxmin_argfilter_workspace_bytes(dtype, batch: int, n: int, w: int) -> int:
    out = ctypes.c_size_t(0)
    _lib.check(_lib.lib().maxmin_argfilter_workspace_bytes(dtype_code(dtype), batch, n, w, ctypes.byref(out)))
    return int(out.value)


def maxmin_argfilter_batched(x: torch.Tensor, w: int, n: int | None = None, *, want_max=True, want_min=True,
                             values=True, workspace=None, stream=None):
    """Arg-max / arg-min filter on every row of a 2-D CUDA tensor [batch, ld] (first n
    columns): returns (out_max, out_min, arg_max, arg_min), positions int64 and absolute
    in the row, ties resolved to the earliest position (N1)."""
    if x.dim() != 2 or not x.is_cuda or x.stride(1) != 1:
        raise ValueError("maxmin_argfilter_batched: x must be a row-major 2-D CUDA tensor")
    batch, ncols = x.shape
    n = ncols if n is None else n
    m = max(n - w + 1, 0)
    out_ld = max((m + 15) // 16 * 16, 16)  # 16-B rows for every output dtype: vector stores
    mk = lambda dt: torch.empty(batch, out_ld, dtype=dt, device=x.device)[:, :m]  # noqa: E731
    out_max = mk(x.dtype) if want_max and values else None
    out_min = mk(x.dtype) if want_min and values else None
    arg_max = mk(torch.int64) if want_max else None
    arg_min = mk(torch.int64) if want_min else None
    need = maxmin_argfilter_workspace_bytes(x.dtype, batch, n, w)
    if workspace is None:
        workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=x.device)
    _lib.check(_lib.lib().maxmin_argfilter_batched(
        dtype_code(x.dtype), _ptr(x), batch, n, x.stride(0), w, _ptr(out_max), _ptr(out_min),
        _ptr(arg_max), _ptr(arg_min), out_ld, _ptr(workspace), workspace.numel() * workspace.element_size(),
        _stream_ptr(stream, x.device)))
    return out_max, out_min, arg_max, arg_min


def maxmin_argfilter_1d(x: torch.Tensor, w: int, **kw):
    """Arg-max / arg-min filter of a contiguous 1-D CUDA tensor (see maxmin_argfilter_batched)."""
    if x.dim() != 1 or not x.is_cuda or not x.is_contiguous():
        raise ValueError("maxmin_argfilter_1d: x must be a contiguous 1-D CUDA tensor")
    outs = maxmin_argfilter_batched(x[None], w, **kw)
    return tuple(o[0] if o is not None else None for o in outs)


def maxmin_lb_keogh_batched(cand: torch.Tensor, query: torch.Tensor, r: int, n: int | None = None, out=None,
                            stream=None):
    """LB_Keogh (N3) of every candidate row of a float32 CUDA tensor [batch, ld] (first n
    columns) against the query (n floats), envelope radius r; returns float64 [batch]."""
    if cand.dim() != 2 or not cand.is_cuda or cand.stride(1) != 1:
        raise ValueError("maxmin_lb_keogh_batched: cand must be a row-major 2-D CUDA tensor")
    batch, ncols = cand.shape
    n = ncols if n is None else n
    if query.dim() != 1 or not query.is_cuda or not query.is_contiguous() or query.shape[0] < n:
        raise ValueError("maxmin_lb_keogh_batched: query must be a contiguous 1-D CUDA tensor of n samples")
    lb = torch.empty(batch, dtype=torch.float64, device=cand.device) if out is None else out
    _lib.check(_lib.lib().maxmin_lb_keogh_batched(dtype_code(cand.dtype), _ptr(cand), batch, n, cand.stride(0),
                                                  _ptr(query), r, _ptr(lb), _stream_ptr(stream, cand.device)))
    return lb


def maxmin_stream_state_bytes(dtype, streams: int, w: int, max_chunk: int) -> int:
    out = ctypes.c_size_t(0)
    _lib.check(_lib.lib().maxmin_stream_state_bytes(dtype_code(dtype), streams, w, max_chunk, ctypes.byref(out)))
    return int(out.value)


class MaxMinStream:
    """Online multi-stream filter (N2): `streams` independent streams with window w.

    ``push(chunk)`` ingests chunk[:, :c] (a [streams, c] CUDA tensor, c <= max_chunk new
    samples per stream) and returns (out_max, out_min, first_valid): column k holds the
    window ending at the k-th new sample; columns < first_valid are not complete windows
    yet (unspecified).  The state lives in one device tensor owned by this object.
    """

    def __init__(self, dtype, streams: int, w: int, max_chunk: int, device=None, stream=None):
        device = torch.device("cuda") if device is None else torch.device(device)
        self.dtype = dtype
        nbytes = maxmin_stream_state_bytes(dtype, streams, w, max_chunk)
        self.state = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)
        self._st = _lib.Stream()
        _lib.check(_lib.lib().maxmin_stream_init(ctypes.byref(self._st), dtype_code(dtype), streams, w, max_chunk,
                                                 _ptr(self.state), nbytes, _stream_ptr(stream, self.state.device)))

    @property
    def seen(self) -> int:
        return int(self._st.seen)

    @property
    def streams(self) -> int:
        return int(self._st.streams)

    @property
    def w(self) -> int:
        return int(self._st.w)

    @property
    def max_chunk(self) -> int:
        return int(self._st.max_chunk)

    def push(self, chunk: torch.Tensor, out_max=None, out_min=None, *, want_max=True, want_min=True,
             stream=None):
        if chunk.dim() != 2 or not chunk.is_cuda or chunk.stride(1) != 1 or chunk.shape[0] != self.streams:
            raise ValueError("MaxMinStream.push: chunk must be a row-major [streams, c] CUDA tensor")
        if chunk.dtype != self.dtype:
            raise TypeError("MaxMinStream.push: chunk dtype differs from the stream's")
        c = chunk.shape[1]
        vec = max(16 // chunk.element_size(), 1)
        c_pad = max((c + vec - 1) // vec * vec, vec)
        _check_out("out_max", out_max, chunk, (self.streams, c))
        _check_out("out_min", out_min, chunk, (self.streams, c))
        _pair_strides("MaxMinStream.push", out_max, out_min, 1)
        if want_max and out_max is None:
            out_max = _alloc_out(out_min, (self.streams, c), self.dtype, chunk.device)
        if want_min and out_min is None:
            out_min = _alloc_out(out_max, (self.streams, c), self.dtype, chunk.device)
        om = out_max if out_max is not None else out_min
        out_ld = om.stride(0) if om is not None else c_pad
        fv = ctypes.c_int64(0)
        _lib.check(_lib.lib().maxmin_stream_push(
            ctypes.byref(self._st), _ptr(chunk), c, chunk.stride(0), _ptr(out_max), _ptr(out_min), out_ld,
            ctypes.byref(fv), _stream_ptr(stream, chunk.device)))
        return out_max, out_min, int(fv.value)


def maxmin_morph_batched(x: torch.Tensor, w: int, n: int | None = None, out_open=None, out_close=None, *,
                         want_open=True, want_close=True, stream=None):
    """Grayscale opening and closing (N4) of every row of a 2-D CUDA tensor [batch, ld] (first
    n columns) by a flat segment of w samples; returns (open, close), each [batch, n]."""
    if x.dim() != 2 or not x.is_cuda or x.stride(1) != 1:
        raise ValueError("maxmin_morph_batched: x must be a row-major 2-D CUDA tensor")
    batch, ncols = x.shape
    n = ncols if n is None else n
    _check_out("out_open", out_open, x, (batch, n))
    _check_out("out_close", out_close, x, (batch, n))
    _pair_strides("maxmin_morph_batched", out_open, out_close, 1)
    if want_open and out_open is None:
        out_open = _alloc_out(out_close, (batch, n), x.dtype, x.device)
    if want_close and out_close is None:
        out_close = _alloc_out(out_open, (batch, n), x.dtype, x.device)
    o = out_open if out_open is not None else out_close
    _lib.check(_lib.lib().maxmin_morph_batched(dtype_code(x.dtype), _ptr(x), batch, n, x.stride(0), w,
                                               _ptr(out_open), _ptr(out_close), o.stride(0) if o is not None else n,
                                               _stream_ptr(stream, x.device)))
    return out_open, out_close


def maxmin_morph_1d(x: torch.Tensor, w: int, **kw):
    """Opening and closing of a contiguous 1-D CUDA tensor (see maxmin_morph_batched)."""
    if x.dim() != 1 or not x.is_cuda or not x.is_contiguous():
        raise ValueError("maxmin_morph_1d: x must be a contiguous 1-D CUDA tensor")
    op, cl = maxmin_morph_batched(x[None], w, **kw)
    return (op[0] if op is not None else None), (cl[0] if cl is not None else None)


def maxmin_morph_2d(x: torch.Tensor, w_row: int, w_col: int, cols: int | None = None, out_open=None,
                    out_close=None, *, want_open=True, want_close=True, workspace=None, stream=None):
    """Opening and closing (N4) of [batch, rows, ld] (or [rows, ld]) images by a flat
    w_col x w_row rectangle; outputs have the images' shape."""
    squeeze = x.dim() == 2
    xx = x[None] if squeeze else x
    if xx.dim() != 3 or not xx.is_cuda or xx.stride(2) != 1:
        raise ValueError("maxmin_morph_2d: x must be a row-major [batch, rows, ld] CUDA tensor")
    batch, rows, ld = xx.shape
    cols = ld if cols is None else cols
    if squeeze:
        out_open = out_open[None] if out_open is not None and out_open.dim() == 2 else out_open
        out_close = out_close[None] if out_close is not None and out_close.dim() == 2 else out_close
    _check_out("out_open", out_open, x, (batch, rows, cols))
    _check_out("out_close", out_close, x, (batch, rows, cols))
    _pair_strides("maxmin_morph_2d", out_open, out_close, 2)
    if want_open and out_open is None:
        out_open = _alloc_out(out_close, (batch, rows, cols), x.dtype, x.device)
    if want_close and out_close is None:
        out_close = _alloc_out(out_open, (batch, rows, cols), x.dtype, x.device)
    o = out_open if out_open is not None else out_close
    need = ctypes.c_size_t(0)
    _lib.check(_lib.lib().maxmin_morph_2d_workspace_bytes(dtype_code(x.dtype), batch, rows, cols, w_row, w_col,
                                                          ctypes.byref(need)))
    if workspace is None:
        workspace = torch.empty(max(need.value, 16), dtype=torch.uint8, device=x.device)
    _lib.check(_lib.lib().maxmin_morph_2d(
        dtype_code(x.dtype), _ptr(xx), batch, rows, cols, xx.stride(1), xx.stride(0), w_row, w_col, _ptr(out_open),
        _ptr(out_close), o.stride(1), o.stride(0), _ptr(workspace), workspace.numel(), _stream_ptr(stream, x.device)))
    if squeeze:
        out_open = out_open[0] if out_open is not None and out_open.dim() == 3 else out_open
        out_close = out_close[0] if out_close is not None and out_close.dim() == 3 else out_close
    return out_open, out_close


def maxmin_filter_3d(x: torch.Tensor, w_x: int, w_y: int, w_z: int, cols: int | None = None, out_max=None,
                     out_min=None, *, want_max=True, want_min=True, workspace=None, stream=None):
    """Max and min over w_z x w_y x w_x boxes of a [depth, rows, ld] CUDA tensor (first `cols`
    columns); outputs [depth-w_z+1, rows-w_y+1, cols-w_x+1] (valid region)."""
    if x.dim() != 3 or not x.is_cuda or x.stride(2) != 1:
        raise ValueError("maxmin_filter_3d: x must be a row-major [depth, rows, ld] CUDA tensor")
    depth, rows, ld = x.shape
    cols = ld if cols is None else cols
    D, R, C = depth - w_z + 1, rows - w_y + 1, cols - w_x + 1
    _check_out("out_max", out_max, x, (max(D, 0), max(R, 0), max(C, 0)))
    _check_out("out_min", out_min, x, (max(D, 0), max(R, 0), max(C, 0)))
    _pair_strides("maxmin_filter_3d", out_max, out_min, 2)
    if want_max and out_max is None and min(D, R, C) > 0:
        out_max = _alloc_out(out_min, (D, R, C), x.dtype, x.device)
    if want_min and out_min is None and min(D, R, C) > 0:
        out_min = _alloc_out(out_max, (D, R, C), x.dtype, x.device)
    o = out_max if out_max is not None else out_min
    need = ctypes.c_size_t(0)
    _lib.check(_lib.lib().maxmin_filter_3d_workspace_bytes(dtype_code(x.dtype), depth, rows, cols, x.stride(1), w_x,
                                                           w_y, w_z, ctypes.byref(need)))
    if workspace is None:
        workspace = torch.empty(max(need.value, 16), dtype=torch.uint8, device=x.device)
    _lib.check(_lib.lib().maxmin_filter_3d(
        dtype_code(x.dtype), _ptr(x), depth, rows, cols, x.stride(1), x.stride(0), w_x, w_y, w_z, _ptr(out_max),
        _ptr(out_min), o.stride(1) if o is not None else C, o.stride(0) if o is not None else R * C, _ptr(workspace),
        workspace.numel(), _stream_ptr(stream, x.device)))
    return out_max, out_min


def maxmin_host_workspace_bytes(dtype, n: int, w: int, chunk: int = 0) -> int:
    out = ctypes.c_size_t(0)
    _lib.check(_lib.lib().maxmin_host_workspace_bytes(dtype_code(dtype), n, w, chunk, ctypes.byref(out)))
    return int(out.value)


def maxmin_filter_1d_host(x: torch.Tensor, w: int, out_max: torch.Tensor, out_min: torch.Tensor,
                          dev_workspace: torch.Tensor, chunk: int = 0) -> None:
    """End-to-end call on HOST (preferably pinned) tensors: H2D, filter, D2H inside."""
    if x.is_cuda or out_max.is_cuda or out_min.is_cuda:
        raise ValueError("maxmin_filter_1d_host: x/out_max/out_min must be host tensors")
    if x.dim() != 1 or not x.is_contiguous():
        raise ValueError("maxmin_filter_1d_host: x must be a contiguous 1-D host tensor")
    m = max(x.shape[0] - w + 1, 0)
    for name, t in (("out_max", out_max), ("out_min", out_min)):
        if t.dtype != x.dtype or t.dim() != 1 or not t.is_contiguous() or t.shape[0] < m:
            raise ValueError(f"maxmin_filter_1d_host: {name} must be a contiguous {x.dtype} host tensor "
                             f"of at least n-w+1 = {m} elements")
    if not dev_workspace.is_cuda:
        raise ValueError("maxmin_filter_1d_host: dev_workspace must be a CUDA tensor")
    need = maxmin_host_workspace_bytes(x.dtype, x.shape[0], w, chunk) if 1 <= w <= x.shape[0] else 0
    if dev_workspace.numel() * dev_workspace.element_size() < need:
        raise ValueError(f"maxmin_filter_1d_host: dev_workspace holds fewer than {need} bytes")
    _lib.check(_lib.lib().maxmin_filter_1d_host(dtype_code(x.dtype), _ptr(x), x.shape[0], w,
                                                _ptr(out_max), _ptr(out_min), chunk,
                                                _ptr(dev_workspace),
                                                dev_workspace.numel() * dev_workspace.element_size()))


def maxmin_sharded_workspace_bytes(dtype, n_local: int, halo: int, windows) -> int:
    ws = (ctypes.c_int64 * len(windows))(*windows)
    out = ctypes.c_size_t(0)
    _lib.check(_lib.lib().maxmin_sharded_workspace_bytes(dtype_code(dtype), n_local, halo, ws, len(windows),
                                                         ctypes.byref(out)))
    return int(out.value)


def maxmin_filter_1d_sharded(local: torch.Tensor, n_local: int, halo: int, windows, out_max, out_min, rank: int,
                             nranks: int, nccl_comm=None, *, workspace=None, stream=None, comm_stream=None):
    """One array split over ranks (include/maxmin.h maxmin_filter_1d_sharded).

    local: 1-D CUDA tensor [own chunk (n_local) | halo slot] (>= n_local + halo elements).
    windows: the windows; out_max / out_min: one CUDA tensor (or None) per window,
    n_local elements (n_local - w + 1 on the last rank).  nccl_comm: the ncclComm_t
    as an int (shard.nccl_comm_ptr), or None when the caller already filled the halo
    slot.  Enqueued on `stream` (NCCL on `comm_stream`); returns immediately."""
    if local.dim() != 1 or not local.is_cuda or not local.is_contiguous() or local.shape[0] < n_local + halo:
        raise ValueError("maxmin_filter_1d_sharded: local must be a contiguous 1-D CUDA tensor of n_local + halo")
    windows = [int(w) for w in windows]
    last = rank == nranks - 1
    for name, outs in (("out_max", out_max), ("out_min", out_min)):
        if len(outs) != len(windows):
            raise ValueError(f"maxmin_filter_1d_sharded: {name} needs one entry per window")
        for w, t in zip(windows, outs):
            _check_out(f"{name}[w={w}]", t, local, (n_local - w + 1 if last else n_local,))
    need = maxmin_sharded_workspace_bytes(local.dtype, n_local, halo, windows)
    if workspace is None and need:
        workspace = torch.empty(need, dtype=torch.uint8, device=local.device)
    wsb = 0 if workspace is None else workspace.numel() * workspace.element_size()
    arr = ctypes.c_int64 * len(windows)
    vps = ctypes.c_void_p * len(windows)
    cs = None if comm_stream is None else ctypes.c_void_p(comm_stream.cuda_stream)
    _lib.check(_lib.lib().maxmin_filter_1d_sharded(
        dtype_code(local.dtype), _ptr(local), n_local, halo, arr(*windows), len(windows), rank, nranks,
        ctypes.c_void_p(nccl_comm or 0), vps(*[t.data_ptr() if t is not None else 0 for t in out_max]),
        vps(*[t.data_ptr() if t is not None else 0 for t in out_min]), _ptr(workspace), wsb,
        _stream_ptr(stream, local.device), cs))
