"""Seeded synthetic inputs shared by the oracle side and the product side.

Holds none of the method's arithmetic: it only writes input arrays.  Heavy
generators are plain C in ``synth/synth.c`` (OpenMP, counter-based SplitMix64,
so every element is a pure function of (seed, stream, index)); the small signal
families of SPEC.md:242-257 used by oracle tests are numpy one-liners here.

Recipes: DESIGN.md section "Inputs"; BASELINE.json configs C1-C5.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynth.so")
_lib = None

# Workload sizes (BASELINE.json:7-11)
C1 = dict(n=100_000, w=16, dtype=np.float64)
C2 = dict(n=1 << 28, windows=(3, 32, 1024, 65536), dtype=np.float32)
C3 = dict(batch=65536, n=4096, w=129, dtype=np.float32)
C4 = dict(batch=8, rows=16384, cols=16384, w_row=15, w_col=15, dtype=np.uint8, nrect=64)
C5 = dict(n=1 << 30, windows=(7, 4096, 262144), dtype=np.float32)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if not force and os.path.exists(_LIB_PATH) and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src):
        return _LIB_PATH
    subprocess.check_call(["gcc", "-O2", "-std=gnu99", "-fopenmp", "-Wall", "-shared", "-fPIC",
                           "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.synth_rng.restype = ctypes.c_uint64
        _lib.synth_c2.restype = ctypes.c_int
        _lib.synth_c5.restype = ctypes.c_int64
    return _lib


def _p(a) -> ctypes.c_void_p:
    """Data pointer of a numpy array or a (CPU) torch tensor."""
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(a.data_ptr())


_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64


def rng(seed: int, stream: int, i: int) -> int:
    return int(_load().synth_rng(_u64(seed), _u64(stream), _u64(i)))


def raw_u64(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    out = np.empty(n, np.uint64)
    _load().synth_raw_u64(_u64(seed), _u64(stream), _i64(offset), _i64(n), _p(out))
    return out


def uniform_f64(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    out = np.empty(n, np.float64)
    _load().synth_uniform_f64(_u64(seed), _u64(stream), _i64(offset), _i64(n), _p(out))
    return out


def uniform_f32(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    out = np.empty(n, np.float32)
    _load().synth_uniform_f32(_u64(seed), _u64(stream), _i64(offset), _i64(n), _p(out))
    return out


def uniform_u8(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    out = np.empty(n, np.uint8)
    _load().synth_uniform_u8(_u64(seed), _u64(stream), _i64(offset), _i64(n), _p(out))
    return out


def normal_f64(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    out = np.empty(n, np.float64)
    _load().synth_normal_f64(_u64(seed), _u64(stream), _i64(offset), _i64(n), _p(out))
    return out


def random_values(dtype, n: int, seed: int, stream: int = 0, alphabet: int | None = None):
    """Seeded values of any supported dtype (full range, or {0..alphabet-1})."""
    dt = np.dtype(dtype)
    raw = raw_u64(seed, stream, n)
    if alphabet is not None:
        return (raw % np.uint64(alphabet)).astype(dt)
    if dt.kind == "f":
        v = uniform_f64(seed, stream, n) * 2.0 - 1.0
        v = v.astype(dt)
        v[v == 0] = 0  # no -0 (BASELINE.json:5)
        return v
    bits = dt.itemsize * 8
    return (raw >> np.uint64(64 - bits)).astype(np.dtype(f"u{dt.itemsize}")).view(dt)


def special_pool(dtype) -> np.ndarray:
    """The values a comparison kernel is most likely to get wrong for a dtype: the
    type's extremes and, for floats, +-inf, subnormals (flushed under FTZ), the
    smallest normals, +-1 and 0 -- never NaN and never -0 (BASELINE.json:5)."""
    dt = np.dtype(dtype)
    if dt.kind == "f":
        fi = np.finfo(dt)
        tiny_sub = np.array(fi.smallest_subnormal, dt)
        v = [-np.inf, np.inf, fi.max, -fi.max, fi.tiny, -fi.tiny, tiny_sub, -tiny_sub, tiny_sub * 7,
             -(tiny_sub * 7), fi.tiny / 2, -(fi.tiny / 2), 0.0, 1.0, -1.0, fi.eps, 1.0 + fi.eps]
        return np.array(v, dt)
    ii = np.iinfo(dt)
    v = {ii.min, ii.max, ii.min + 1, ii.max - 1, 0, 1}
    if ii.min < 0:
        v.add(-1)
    return np.array(sorted(v), dt)


def edge_values(dtype, n: int, seed: int, stream: int = 0) -> np.ndarray:
    """Seeded edge-case series: runs of values drawn from special_pool(dtype) (run
    lengths 1..64, and every 7th run 500..3000 long: long equal runs), mixed with
    runs of ordinary random values of the dtype."""
    dt = np.dtype(dtype)
    pool = special_pool(dt)
    raw = raw_u64(seed, stream, 4 * (n // 8 + 16))
    ordinary = random_values(dt, n, seed + 1, stream)
    out = np.empty(n, dt)
    i = k = 0
    while i < n:
        r = int(raw[k % raw.shape[0]]); k += 1
        length = 500 + r % 2500 if k % 7 == 0 else 1 + (r >> 8) % 64
        length = min(length, n - i)
        if (r >> 20) % 4 == 0:  # a run of ordinary values
            out[i:i + length] = ordinary[i:i + length]
        elif (r >> 20) % 4 == 1:  # distinct specials, one per position
            idx = raw[(k + np.arange(length)) % raw.shape[0]] % np.uint64(pool.shape[0])
            out[i:i + length] = pool[idx.astype(np.int64)]
        else:  # a constant run of one special
            out[i:i + length] = pool[(r >> 24) % pool.shape[0]]
        i += length
    if dt.kind == "f":
        out[out == 0] = 0  # no -0
    return out


# ---- BASELINE workloads -----------------------------------------------------

def c1(out=None) -> np.ndarray:
    out = np.empty(C1["n"], np.float64) if out is None else out
    _load().synth_c1(_i64(out.shape[0]), _p(out))
    return out


def c2(n: int = C2["n"], stream: int = 0, out=None):
    """Random walk of length n; ``out`` may be a numpy array or pinned torch tensor."""
    out = np.empty(n, np.float32) if out is None else out
    rc = _load().synth_c2(_u64(stream), _i64(n), _p(out))
    if rc != 0:
        raise MemoryError("synth_c2")
    return out


def c3(rows: int = C3["batch"], row0: int = 0, length: int = C3["n"], ld: int | None = None, out=None):
    ld = length if ld is None else ld
    out = np.empty((rows, ld), np.float32) if out is None else out
    _load().synth_c3(_i64(row0), _i64(rows), _i64(length), _i64(ld), _p(out))
    return out


def c4(count: int = C4["batch"], img0: int = 0, rows: int = C4["rows"], cols: int = C4["cols"],
       ld: int | None = None, nrect: int = C4["nrect"], out=None):
    ld = cols if ld is None else ld
    out = np.empty((count, rows, ld), np.uint8) if out is None else out
    _load().synth_c4(_i64(img0), _i64(count), _i64(rows), _i64(cols), _i64(ld), ctypes.c_int(nrect),
                     _p(out))
    return out


def c5(n: int = C5["n"], stream: int = 0, out=None):
    out = np.empty(n, np.float32) if out is None else out
    rc = _load().synth_c5(_u64(stream), _i64(n), _p(out))
    if rc < 0:
        raise MemoryError("synth_c5")
    return out


# ---- SPEC.md:242-257 signal families (small, for oracle pins) ---------------

def sine(n: int, period: float) -> np.ndarray:
    v = np.sin(2.0 * np.pi * np.arange(n) / period)
    v[v == 0] = 0.0
    return v


def ramp_up(n: int) -> np.ndarray:
    return np.arange(n, dtype=np.float64)


def ramp_down(n: int) -> np.ndarray:
    return np.arange(n, 0, -1, dtype=np.float64)


def constant(n: int, level: float = 7.0) -> np.ndarray:
    return np.full(n, level, np.float64)


def alternating(n: int) -> np.ndarray:
    return (np.arange(n) % 2).astype(np.float64)


def piecewise(n: int, segments: int, seed: int) -> np.ndarray:
    """Concatenated seeded monotone segments (alternately rising and falling)."""
    cuts = np.sort(raw_u64(seed, 7, max(segments - 1, 0)) % np.uint64(max(n, 1))).astype(np.int64)
    bounds = np.concatenate([[0], cuts, [n]])
    out = np.empty(n, np.float64)
    base = uniform_f64(seed, 8, segments + 1) * 100.0
    for s in range(len(bounds) - 1):
        b, e = bounds[s], bounds[s + 1]
        t = np.arange(e - b, dtype=np.float64)
        out[b:e] = base[s] + (t if s % 2 == 0 else -t)
    out[out == 0] = 0.0
    return out
