"""CPU oracle for the running max-min filter (arXiv cs/0610046).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product package ``paper_cs_0610046_b200`` never imports it and
shares no code with it.

Thin ctypes marshalling over ``liboracle.so`` (plain C, ``oracle/oracle.c`` +
``oracle/oracle_body.inc``).  Every arithmetic step lives in the C file and
cites the PAPER.md passage it follows:

=====================  ====================================================
``brute_1d``           definition; Table 1 naive, PAPER.md:135
``alg1``               Algorithm 1, PAPER.md:364-401 (readings R1-R4)
``appendix``           appendix listing
``w3``                 Proposition (w = 3)
``vhgw``               van Herk-Gil-Werman, PAPER.md:108-116, 176-192 (R7)
``brute_2d``           2-D rectangle definition, valid region (R9)
``separable_2d``       rows then columns, PAPER.md:61-63
``batched``            ``appendix`` on every row
``windows_at``         brute force at a list of window starts
``arg_brute/arg_wedge`` N1 arg filter (definition / wedge keeping ties, R17)
``keogh``              N3 LB_Keogh (clipped envelope, R18)
``Stream``             N2 one stream's wedge, zero-latency pushes (R19)
``morph`` / ``morph_2d`` N4 opening and closing (definition or composition, R20)
``brute_3d`` / ``separable_3d`` N4 N-D separable filter: 3-D boxes (definition / axis by axis)
=====================  ====================================================

Parity pins live in ``tests/test_oracle_*.py``; none of the functions is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

_SUFFIX = {
    np.dtype(np.uint8): "u8",
    np.dtype(np.int8): "i8",
    np.dtype(np.uint16): "u16",
    np.dtype(np.int16): "i16",
    np.dtype(np.uint32): "u32",
    np.dtype(np.int32): "i32",
    np.dtype(np.uint64): "u64",
    np.dtype(np.int64): "i64",
    np.dtype(np.float32): "f32",
    np.dtype(np.float64): "f64",
}
DTYPES = tuple(_SUFFIX)

_ERRORS = {
    -1: "window < 1 (or not 3 for w3)",
    -2: "window larger than input",
    -3: "NaN in input",
    -4: "paper invariant violated (deque capacity)",
    -5: "allocation failure",
    -6: "bad shape",
}


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle error {code}: {_ERRORS.get(code, 'unknown')}")
        self.code = code


class _Stats(ctypes.Structure):
    _fields_ = [("comparisons", ctypes.c_uint64), ("peak_wedge", ctypes.c_int64)]


@dataclass
class Stats:
    comparisons: int
    peak_wedge: int


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, IEEE-exact: no fast-math)."""
    src = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "oracle_body.inc"),
           os.path.join(_HERE, "oracle.h")]
    if not force and os.path.exists(_LIB_PATH):
        if os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(s) for s in src):
            return _LIB_PATH
    subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC", "-o",
                           _LIB_PATH, src[0], "-lm"])
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------- CPU baseline
# The same C sources built with -O3 -march=native, used ONLY to time the oracle
# as the CPU baseline ("O3 built with g++ -O3
# -march=native", one thread and all host threads).  -march=native binds the
# build to the host it runs on, so it is compiled there, on first use.
_NATIVE_PATH = os.path.join(_HERE, "liboracle_native.so")
_native = None
NATIVE_FLAGS = ["-O3", "-march=native"]


def build_native(force: bool = False) -> str:
    src = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "oracle_body.inc"),
           os.path.join(_HERE, "oracle.h")]
    if not force and os.path.exists(_NATIVE_PATH):
        if os.path.getmtime(_NATIVE_PATH) >= max(os.path.getmtime(s) for s in src):
            return _NATIVE_PATH
    tmp = _NATIVE_PATH + f".{os.getpid()}.tmp"
    subprocess.check_call(["gcc", *NATIVE_FLAGS, "-std=c99", "-Wall", "-shared", "-fPIC", "-o", tmp, src[0], "-lm"])
    os.replace(tmp, _NATIVE_PATH)
    return _NATIVE_PATH


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def appendix_baseline(a, w: int, threads: int = 1, out_max=None, out_min=None):
    """The appendix listing from the -O3 -march=native build,
    on `threads` host threads: the m windows are cut into contiguous ranges, each
    range filtered from its own input slice (the range plus w-1 elements of
    overlap) by one sequential call.  ctypes releases the GIL during the calls,
    so the threads run in parallel.  Returns (max, min)."""
    global _native
    if _native is None:
        build_native()
        _native = ctypes.CDLL(_NATIVE_PATH)
    a = np.ascontiguousarray(a)
    n = a.shape[0]
    m = n - w + 1
    if m <= 0:
        raise OracleError(-2)
    mx = np.empty(m, a.dtype) if out_max is None else out_max
    mn = np.empty(m, a.dtype) if out_min is None else out_min
    f = getattr(_native, f"oracle_appendix_{_SUFFIX[a.dtype]}")
    f.restype = ctypes.c_int
    sz = a.dtype.itemsize
    threads = max(1, min(threads, m))
    bounds = [m * k // threads for k in range(threads + 1)]

    def run(k):
        j0, j1 = bounds[k], bounds[k + 1]
        if j1 <= j0:
            return 0
        st = _Stats()
        return f(ctypes.c_void_p(a.ctypes.data + j0 * sz), ctypes.c_int64(j1 - j0 + w - 1), ctypes.c_int64(w),
                 ctypes.c_void_p(mx.ctypes.data + j0 * sz), ctypes.c_void_p(mn.ctypes.data + j0 * sz),
                 ctypes.byref(st))

    if threads == 1:
        _check(run(0))
    else:
        import concurrent.futures as cf

        with cf.ThreadPoolExecutor(max_workers=threads) as ex:
            for rc in ex.map(run, range(threads)):
                _check(rc)
    return mx, mn


def _fn(name: str, dtype):
    dt = np.dtype(dtype)
    if dt not in _SUFFIX:
        raise TypeError(f"oracle: unsupported dtype {dt}")
    f = getattr(_load(), f"oracle_{name}_{_SUFFIX[dt]}")
    f.restype = ctypes.c_int
    return f


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc)


def _run_1d(name: str, a, w: int):
    a = np.ascontiguousarray(a)
    n = a.shape[0]
    m = max(n - w + 1, 0)
    mx = np.empty(m, a.dtype)
    mn = np.empty(m, a.dtype)
    st = _Stats()
    _check(_fn(name, a.dtype)(_ptr(a), ctypes.c_int64(n), ctypes.c_int64(w), _ptr(mx),
                              _ptr(mn), ctypes.byref(st)))
    return mx, mn, Stats(int(st.comparisons), int(st.peak_wedge))


def _run_arg(name: str, a, w: int):
    a = np.ascontiguousarray(a)
    n = a.shape[0]
    m = max(n - w + 1, 0)
    mx, mn = np.empty(m, a.dtype), np.empty(m, a.dtype)
    ax, an = np.empty(m, np.int64), np.empty(m, np.int64)
    _check(_fn(name, a.dtype)(_ptr(a), ctypes.c_int64(n), ctypes.c_int64(w), _ptr(mx), _ptr(mn),
                              _ptr(ax), _ptr(an)))
    return mx, mn, ax, an


def arg_brute(a, w: int):
    """N1 arg filter, the definition: (max, min, argmax, argmin), earliest positions."""
    return _run_arg("arg_brute", a, w)


def arg_wedge(a, w: int):
    """N1 arg filter by the paper's wedge with equal values kept (earliest positions)."""
    return _run_arg("arg_wedge", a, w)


def keogh(c, q, r: int, brute: bool = False, envelope: bool = False):
    """N3 LB_Keogh of every candidate row of c [batch, n] against the query q [n] with
    warping radius r (float32 data, float64 bounds).  With envelope=True also returns
    the clipped envelope (U, L) as [batch, n] float32 arrays."""
    c = np.ascontiguousarray(c, dtype=np.float32)
    if c.ndim == 1:
        c = c[None]
    q = np.ascontiguousarray(q, dtype=np.float32)
    batch, n = c.shape
    lb = np.empty(batch, np.float64)
    U = np.empty((batch, n), np.float32) if envelope else None
    L = np.empty((batch, n), np.float32) if envelope else None
    f = getattr(_load(), "oracle_keogh_brute_f32" if brute else "oracle_keogh_f32")
    f.restype = ctypes.c_int
    _check(f(_ptr(c), ctypes.c_int64(batch), ctypes.c_int64(n), ctypes.c_int64(n), _ptr(q), ctypes.c_int64(r),
             _ptr(lb), ctypes.c_void_p(None) if U is None else _ptr(U),
             ctypes.c_void_p(None) if L is None else _ptr(L)))
    return (lb, U, L) if envelope else lb


def brute_1d(a, w: int):
    """O1, the definition.  Returns (max, min, Stats)."""
    return _run_1d("brute_1d", a, w)


def alg1(a, w: int):
    """O2, Algorithm 1 read literally.  w >= 2."""
    return _run_1d("alg1", a, w)


def appendix(a, w: int):
    """O3, the appendix C++ listing.  w >= 1."""
    return _run_1d("appendix", a, w)


def vhgw(a, w: int):
    """van Herk-Gil-Werman baseline."""
    return _run_1d("vhgw", a, w)


def w3(a):
    """Proposition w = 3."""
    a = np.ascontiguousarray(a)
    n = a.shape[0]
    m = max(n - 2, 0)
    mx = np.empty(m, a.dtype)
    mn = np.empty(m, a.dtype)
    st = _Stats()
    _check(_fn("w3", a.dtype)(_ptr(a), ctypes.c_int64(n), _ptr(mx), _ptr(mn),
                              ctypes.byref(st)))
    return mx, mn, Stats(int(st.comparisons), int(st.peak_wedge))


def batched(a, w: int, n: int | None = None):
    """``appendix`` on every row of a 2-D array ``a[batch, ld]`` (first n columns)."""
    a = np.ascontiguousarray(a)
    batch, ld = a.shape
    n = ld if n is None else n
    m = n - w + 1
    mx = np.empty((batch, max(m, 0)), a.dtype)
    mn = np.empty((batch, max(m, 0)), a.dtype)
    _check(_fn("batched", a.dtype)(_ptr(a), ctypes.c_int64(batch), ctypes.c_int64(n),
                                   ctypes.c_int64(ld), ctypes.c_int64(w), _ptr(mx), _ptr(mn),
                                   ctypes.c_int64(max(m, 1))))
    return mx, mn


def _run_2d(name: str, a, w_row: int, w_col: int):
    a = np.ascontiguousarray(a)
    squeeze = a.ndim == 2
    if squeeze:
        a = a[None]
    batch, rows, cols = a.shape
    R, C = rows - w_col + 1, cols - w_row + 1
    mx = np.empty((batch, max(R, 0), max(C, 0)), a.dtype)
    mn = np.empty_like(mx)
    _check(_fn(name, a.dtype)(_ptr(a), ctypes.c_int64(batch), ctypes.c_int64(rows),
                              ctypes.c_int64(cols), ctypes.c_int64(w_row), ctypes.c_int64(w_col),
                              _ptr(mx), _ptr(mn)))
    if squeeze:
        return mx[0], mn[0]
    return mx, mn


def brute_2d(a, w_row: int, w_col: int):
    """2-D rectangle max/min over the valid region (reading R9)."""
    return _run_2d("brute_2d", a, w_row, w_col)


def separable_2d(a, w_row: int, w_col: int):
    """Rows first, then columns, ``appendix`` as the 1-D filter."""
    return _run_2d("separable_2d", a, w_row, w_col)


def windows_at(a, w: int, starts):
    """Brute-force max/min of the windows starting at ``starts`` (spot checks)."""
    a = np.ascontiguousarray(a)
    starts = np.ascontiguousarray(starts, dtype=np.int64)
    mx = np.empty(starts.shape[0], a.dtype)
    mn = np.empty(starts.shape[0], a.dtype)
    _check(_fn("windows_at", a.dtype)(_ptr(a), ctypes.c_int64(a.shape[0]), ctypes.c_int64(w),
                                      _ptr(starts), ctypes.c_int64(starts.shape[0]), _ptr(mx),
                                      _ptr(mn)))
    return mx, mn


class Stream:
    """N2: one stream's monotonic wedge (Algorithm 1), fed by pushes
    of any length; every window is returned by the push of its last sample (R19)."""

    def __init__(self, dtype, w: int):
        self.dtype = np.dtype(dtype)
        self.w = w
        self._h = ctypes.c_void_p()
        _check(_fn("stream_new", self.dtype)(ctypes.c_int64(w), ctypes.byref(self._h)))
        self._push = _fn("stream_push", self.dtype)

    def push(self, x):
        """Ingest the samples x; returns (max, min) of the windows they complete."""
        x = np.ascontiguousarray(x, dtype=self.dtype)
        c = x.shape[0]
        mx, mn = np.empty(c, self.dtype), np.empty(c, self.dtype)
        e = ctypes.c_int64(0)
        _check(self._push(self._h, _ptr(x) if c else ctypes.c_void_p(None), ctypes.c_int64(c), _ptr(mx), _ptr(mn),
                          ctypes.byref(e)))
        return mx[:e.value], mn[:e.value]

    def stats(self) -> Stats:
        st = _Stats()
        f = _load().oracle_stream_stats
        f.restype = ctypes.c_int
        _check(f(self._h, ctypes.byref(st)))
        return Stats(int(st.comparisons), int(st.peak_wedge))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.oracle_stream_free(h)
            self._h = ctypes.c_void_p()


def stream_pushes(rows, w: int, sizes):
    """N2 on many streams: rows [S, N] pushed in chunks of the given sizes (summing to
    <= N); returns per push (out_max [S, e], out_min [S, e]) of the windows completed."""
    rows = np.ascontiguousarray(rows)
    streams = [Stream(rows.dtype, w) for _ in range(rows.shape[0])]
    res, off = [], 0
    for c in sizes:
        outs = [s.push(rows[i, off:off + c]) for i, s in enumerate(streams)]
        res.append((np.stack([o[0] for o in outs]) if outs else np.empty((0, 0), rows.dtype),
                    np.stack([o[1] for o in outs]) if outs else np.empty((0, 0), rows.dtype)))
        off += c
    return res


def morph(a, w: int, brute: bool = False):
    """N4 grayscale (opening, closing) of a 1-D array by a flat segment of w samples
    (reading R20); brute=True evaluates the definition, else the composition."""
    a = np.ascontiguousarray(a)
    n = a.shape[0]
    op, cl = np.empty(n, a.dtype), np.empty(n, a.dtype)
    _check(_fn("morph_brute" if brute else "morph", a.dtype)(_ptr(a), ctypes.c_int64(n), ctypes.c_int64(w),
                                                             _ptr(op), _ptr(cl)))
    return op, cl


def morph_2d(a, w_row: int, w_col: int, brute: bool = False):
    """N4 (opening, closing) of [batch,] rows x cols images by a flat w_col x w_row rectangle."""
    a = np.ascontiguousarray(a)
    squeeze = a.ndim == 2
    if squeeze:
        a = a[None]
    batch, rows, cols = a.shape
    op, cl = np.empty_like(a), np.empty_like(a)
    _check(_fn("morph_2d_brute" if brute else "morph_2d", a.dtype)(
        _ptr(a), ctypes.c_int64(batch), ctypes.c_int64(rows), ctypes.c_int64(cols), ctypes.c_int64(w_row),
        ctypes.c_int64(w_col), _ptr(op), _ptr(cl)))
    return (op[0], cl[0]) if squeeze else (op, cl)


def _run_3d(name: str, a, w_x: int, w_y: int, w_z: int):
    a = np.ascontiguousarray(a)
    depth, rows, cols = a.shape
    D, R, C = depth - w_z + 1, rows - w_y + 1, cols - w_x + 1
    mx = np.empty((max(D, 0), max(R, 0), max(C, 0)), a.dtype)
    mn = np.empty_like(mx)
    _check(_fn(name, a.dtype)(_ptr(a), ctypes.c_int64(depth), ctypes.c_int64(rows), ctypes.c_int64(cols),
                              ctypes.c_int64(w_x), ctypes.c_int64(w_y), ctypes.c_int64(w_z), _ptr(mx), _ptr(mn)))
    return mx, mn


def brute_3d(a, w_x: int, w_y: int, w_z: int):
    """3-D max/min over w_z x w_y x w_x boxes, valid region (the definition)."""
    return _run_3d("brute_3d", a, w_x, w_y, w_z)


def separable_3d(a, w_x: int, w_y: int, w_z: int):
    """The 1-D filter along columns, rows, then depth (PAPER.md:61-63 extended)."""
    return _run_3d("separable_3d", a, w_x, w_y, w_z)
