"""Seeded randomized sweep of every C-ABI entry point (include/maxmin.h) on the GPU.

Each case draws a dtype, a shape, a window and a memory layout -- base offsets in
elements, row / image pitches with padding -- and calls the library through ctypes
with exactly those pointers.  The layout rules of the header predict the status:
a layout the header allows must return MAXMIN_OK and match the oracle bit for bit
(LB_Keogh: relative 1e-12, reading R18); a layout it forbids must return
MAXMIN_ERR_ALIGNMENT and leave the outputs untouched.  Windows are drawn from every
kernel path's range (log-step, lane-group, large-window look-back).
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_cs_0610046_b200")

DEV = torch.device("cuda:0")
VP = ctypes.c_void_p
ALL = [np.uint8, np.int8, np.uint16, np.int16, np.uint32, np.int32, np.uint64, np.int64, np.float32, np.float64]
ARG = [np.uint8, np.int8, np.uint16, np.int16, np.uint32, np.int32, np.float32]
OK, ALIGN = 0, 6
SENTINEL = 0x5A


def _tdt(dtype):
    return torch.from_numpy(np.zeros(1, dtype)).dtype


def _code(dtype):
    return mm.dtype_code(_tdt(dtype))


def _stream():
    return VP(torch.cuda.current_stream().cuda_stream)


class Buf:
    """A device buffer holding `rows` rows of `n` elements at pitch `ld`, starting
    `off` elements past a 256-byte aligned allocation (bytes outside the rows keep
    a sentinel, so stray writes show)."""

    def __init__(self, dtype, rows, n, ld, off, host=None):
        self.dt = np.dtype(dtype)
        self.rows, self.n, self.ld, self.off = rows, n, ld, off
        total = off + (rows - 1) * ld + n if rows > 0 else off + 1
        self.t = torch.full((total * self.dt.itemsize + 64,), SENTINEL, dtype=torch.uint8, device=DEV)
        if host is not None:
            full = np.frombuffer(self.t.cpu().numpy().tobytes(), dtype=np.uint8).copy()
            view = full[: total * self.dt.itemsize].view(self.dt)
            for r in range(rows):
                view[off + r * ld: off + r * ld + n] = host[r]
            self.t.copy_(torch.from_numpy(full))

    @property
    def ptr(self):
        return VP(self.t.data_ptr() + self.off * self.dt.itemsize)

    def rows_np(self):
        full = self.t.cpu().numpy()
        total = self.off + (self.rows - 1) * self.ld + self.n
        view = full[: total * self.dt.itemsize].view(self.dt)
        return np.stack([view[self.off + r * self.ld: self.off + r * self.ld + self.n] for r in range(self.rows)])

    def untouched(self):
        return bool((self.t.cpu().numpy() == SENTINEL).all())


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.dtype(f"u{a.dtype.itemsize}"))


def _same(got, exp, what):
    g, e = _bits(got), _bits(exp)
    assert g.shape == e.shape, (what, g.shape, e.shape)
    if not np.array_equal(g, e):
        bad = np.flatnonzero((g != e).ravel())
        raise AssertionError(f"{what}: {bad.size} mismatches, first at {bad[0]}")


def _values(dtype, n, seed):
    k = seed % 3
    if k == 0:
        return synth.random_values(dtype, n, seed=seed)
    if k == 1:
        return synth.random_values(dtype, n, seed=seed, alphabet=5)  # ties
    return synth.edge_values(dtype, n, seed=seed)


def _n(rng, lo=1, hi=60000):
    return int(np.exp(rng.uniform(np.log(lo), np.log(hi))))


def _shape(rng, cap=None, m_hi=60000):
    """(n, w): a window from one of the kernel paths' ranges (log-step, lane-group,
    look-back), then n = w - 1 + m with m log-uniform (ragged tails, single outputs)."""
    lo, hi = [(1, 16), (17, 300), (301, 1024), (1025, 8193), (8194, 70000)][rng.integers(0, 5)]
    if cap is not None:
        hi = min(hi, cap)
        lo = min(lo, hi)
    w = int(rng.integers(lo, hi + 1))
    return w - 1 + _n(rng, 1, m_hi), w


# ------------------------------------------------------------------ 1-D batched

@pytest.mark.parametrize("case", range(240))
def test_fuzz_batched(cuda_device, case):
    rng = np.random.default_rng(1000 + case)
    dtype = ALL[case % len(ALL)]
    sz = np.dtype(dtype).itemsize
    batch = int(rng.choice([1, 1, 2, 3, 5]))
    n, w = _shape(rng)
    m = n - w + 1
    vec = 16 // sz
    aligned = rng.random() < 0.8
    in_off = 0 if aligned else int(rng.integers(1, vec + 1))
    in_ld = (n + vec - 1) // vec * vec + int(rng.integers(0, 3)) * vec if aligned else n + int(rng.integers(0, 5))
    out_ld = (m + vec - 1) // vec * vec + int(rng.integers(0, 2)) * vec if aligned else m + int(rng.integers(0, 5))
    out_off = 0 if (aligned or rng.random() < 0.5) else int(rng.integers(1, vec + 1))
    a = _values(dtype, batch * n, 1000 + case).reshape(batch, n)
    x = Buf(dtype, batch, n, in_ld, in_off, a)
    ox = Buf(dtype, batch, m, out_ld, out_off)
    on = Buf(dtype, batch, m, out_ld, out_off)
    need = mm.maxmin_workspace_bytes(_tdt(dtype), batch, n, w)
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device=DEV)
    ok_layout = ((in_off * sz) % 16 == 0 and (out_off * sz) % 16 == 0 and
                 (batch == 1 or ((in_ld * sz) % 16 == 0 and (out_ld * sz) % 16 == 0)))
    rc = mm._lib.lib().maxmin_filter_batched(_code(dtype), x.ptr, batch, n, in_ld, w, ox.ptr, on.ptr, out_ld,
                                             VP(ws.data_ptr()), need, _stream())
    torch.cuda.synchronize()
    what = f"{np.dtype(dtype).name} batch={batch} n={n} w={w} in=({in_off},{in_ld}) out=({out_off},{out_ld})"
    if not ok_layout:
        assert rc == ALIGN, what
        assert ox.untouched() and on.untouched(), what
        return
    assert rc == OK, (what, rc)
    ex, en = oracle.batched(a, w)
    _same(ox.rows_np(), ex, "max " + what)
    _same(on.rows_np(), en, "min " + what)


# ------------------------------------------------------------------------- 2-D

@pytest.mark.parametrize("case", range(160))
def test_fuzz_2d(cuda_device, case):
    rng = np.random.default_rng(2000 + case)
    dtype = ALL[case % len(ALL)]
    batch = int(rng.integers(1, 4))
    rows, cols = _n(rng, 1, 260), _n(rng, 1, 700)
    if np.dtype(dtype).itemsize == 1 and rng.random() < 0.5:  # the packed-byte kernel's domain
        wr = wc = int(rng.integers(1, min(17, rows, cols) + 1))
    else:
        wr, wc = int(rng.integers(1, min(cols, 40) + 1)), int(rng.integers(1, min(rows, 40) + 1))
    R, C = rows - wc + 1, cols - wr + 1
    in_off, in_ld = int(rng.integers(0, 5)), cols + int(rng.integers(0, 9))
    in_bs = rows * in_ld + int(rng.integers(0, 7))
    out_off, out_ld = int(rng.integers(0, 5)), C + int(rng.integers(0, 9))
    out_bs = R * out_ld + int(rng.integers(0, 7))
    img = _values(dtype, batch * rows * cols, 2000 + case).reshape(batch, rows, cols)
    # the images as one flat run of elements: row r of image b at b*in_bs + r*in_ld
    total = (batch - 1) * in_bs + (rows - 1) * in_ld + cols
    host = np.zeros(total, dtype)
    for b in range(batch):
        for r in range(rows):
            host[b * in_bs + r * in_ld: b * in_bs + r * in_ld + cols] = img[b, r]
    x = Buf(dtype, 1, total, total, in_off, host[None])
    span = (batch - 1) * out_bs + (R - 1) * out_ld + C
    ox, on = Buf(dtype, 1, span, span, out_off), Buf(dtype, 1, span, span, out_off)
    need = ctypes.c_size_t(0)
    L = mm._lib.lib()
    assert L.maxmin_filter_2d_workspace_bytes(_code(dtype), batch, rows, cols, wr, wc, ctypes.byref(need)) == OK
    ws = torch.empty(max(need.value, 16), dtype=torch.uint8, device=DEV)
    rc = L.maxmin_filter_2d_ws(_code(dtype), x.ptr, batch, rows, cols, in_ld, in_bs, wr, wc, ox.ptr, on.ptr, out_ld,
                               out_bs, VP(ws.data_ptr()), ws.numel(), _stream())
    torch.cuda.synchronize()
    what = f"{np.dtype(dtype).name} {batch}x{rows}x{cols} w={wr}x{wc} in=({in_off},{in_ld},{in_bs}) " \
           f"out=({out_off},{out_ld},{out_bs})"
    assert rc == OK, (what, rc)
    gx, gn = ox.rows_np()[0], on.rows_np()[0]
    for b in range(batch):
        ex, en = oracle.separable_2d(img[b], wr, wc)
        for src, exp, nm in ((gx, ex, "max"), (gn, en, "min")):
            got = np.stack([src[b * out_bs + r * out_ld: b * out_bs + r * out_ld + C] for r in range(R)])
            _same(got, exp, f"{nm} image {b} " + what)


# ------------------------------------------------------------------ arg filter

@pytest.mark.parametrize("case", range(112))
def test_fuzz_argfilter(cuda_device, case):
    rng = np.random.default_rng(3000 + case)
    dtype = ARG[case % len(ARG)]
    batch = int(rng.choice([1, 1, 2, 3]))
    n, w = _shape(rng, cap=20000, m_hi=20000)
    m = n - w + 1
    in_off, in_ld = int(rng.integers(0, 5)), n + int(rng.integers(0, 6))
    out_off, out_ld = int(rng.integers(0, 5)), m + int(rng.integers(0, 6))
    a = _values(dtype, batch * n, 3000 + case).reshape(batch, n)
    x = Buf(dtype, batch, n, in_ld, in_off, a)
    ox, on = Buf(dtype, batch, m, out_ld, out_off), Buf(dtype, batch, m, out_ld, out_off)
    ax, an = Buf(np.int64, batch, m, out_ld, out_off), Buf(np.int64, batch, m, out_ld, out_off)
    need = mm.maxmin_argfilter_workspace_bytes(_tdt(dtype), batch, n, w)
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device=DEV)
    rc = mm._lib.lib().maxmin_argfilter_batched(_code(dtype), x.ptr, batch, n, in_ld, w, ox.ptr, on.ptr, ax.ptr,
                                                an.ptr, out_ld, VP(ws.data_ptr()), need, _stream())
    torch.cuda.synchronize()
    what = f"{np.dtype(dtype).name} batch={batch} n={n} w={w} in=({in_off},{in_ld}) out=({out_off},{out_ld})"
    assert rc == OK, (what, rc)
    gx, gn, gax, gan = ox.rows_np(), on.rows_np(), ax.rows_np(), an.rows_np()
    for r in range(batch):
        ex, en, eax, ean = oracle.arg_wedge(a[r], w)
        _same(gx[r], ex, f"row {r} max " + what)
        _same(gn[r], en, f"row {r} min " + what)
        _same(gax[r], eax, f"row {r} argmax " + what)
        _same(gan[r], ean, f"row {r} argmin " + what)


# ------------------------------------------------------------------ morphology

@pytest.mark.parametrize("case", range(120))
def test_fuzz_morph(cuda_device, case):
    rng = np.random.default_rng(4000 + case)
    dtype = ALL[case % len(ALL)]
    sz = np.dtype(dtype).itemsize
    vec = 16 // sz
    batch = int(rng.choice([1, 1, 2, 4]))
    n, w = _shape(rng, cap=3000 if sz == 8 else 8193, m_hi=20000)
    in_off, in_ld = int(rng.integers(0, 5)), n + int(rng.integers(0, 6))
    aligned = rng.random() < 0.85
    out_off = 0 if aligned else int(rng.integers(1, vec + 1))
    out_ld = (n + vec - 1) // vec * vec if aligned else n + int(rng.integers(0, 4))
    a = _values(dtype, batch * n, 4000 + case).reshape(batch, n)
    x = Buf(dtype, batch, n, in_ld, in_off, a)
    oo, oc = Buf(dtype, batch, n, out_ld, out_off), Buf(dtype, batch, n, out_ld, out_off)
    ok_layout = (out_off * sz) % 16 == 0 and (batch == 1 or (out_ld * sz) % 16 == 0)
    rc = mm._lib.lib().maxmin_morph_batched(_code(dtype), x.ptr, batch, n, in_ld, w, oo.ptr, oc.ptr, out_ld,
                                            _stream())
    torch.cuda.synchronize()
    what = f"{np.dtype(dtype).name} batch={batch} n={n} w={w} in=({in_off},{in_ld}) out=({out_off},{out_ld})"
    if not ok_layout:
        assert rc == ALIGN, what
        assert oo.untouched() and oc.untouched(), what
        return
    assert rc == OK, (what, rc)
    go, gc = oo.rows_np(), oc.rows_np()
    for r in range(batch):
        eo, ec = oracle.morph(a[r], w)
        _same(go[r], eo, f"row {r} open " + what)
        _same(gc[r], ec, f"row {r} close " + what)


# -------------------------------------------------------------------- LB_Keogh

@pytest.mark.parametrize("case", range(48))
def test_fuzz_keogh(cuda_device, case):
    rng = np.random.default_rng(5000 + case)
    batch = int(rng.integers(1, 6))
    n = _n(rng, 1, 20000)
    r = int(rng.choice([0, int(rng.integers(1, 40)), int(rng.integers(40, 4096)), n + int(rng.integers(0, 9))]))
    ld = (n + 3) // 4 * 4 + 4 * int(rng.integers(0, 3))
    q_off = int(rng.integers(0, 4))
    c = synth.random_values(np.float32, batch * n, seed=5000 + case).reshape(batch, n)
    qv = synth.random_values(np.float32, n, seed=5100 + case)
    x = Buf(np.float32, batch, n, ld, 0, c)
    q = Buf(np.float32, 1, n, n, q_off, qv[None])
    lb = torch.empty(batch, dtype=torch.float64, device=DEV)
    rc = mm._lib.lib().maxmin_lb_keogh_batched(_code(np.float32), x.ptr, batch, n, ld, q.ptr, r,
                                               VP(lb.data_ptr()), _stream())
    torch.cuda.synchronize()
    what = f"batch={batch} n={n} r={r} ld={ld} q_off={q_off}"
    assert rc == OK, (what, rc)
    exp = oracle.keogh(c, qv, r)
    got = lb.cpu().numpy()
    assert np.all(np.abs(got - exp) <= 1e-12 * np.maximum(1.0, np.abs(exp))), what


# ---------------------------------------------------------------- stream pushes

@pytest.mark.parametrize("case", range(60))
def test_fuzz_stream(cuda_device, case):
    rng = np.random.default_rng(6000 + case)
    dtype = ALL[case % len(ALL)]
    S = int(rng.integers(1, 40))
    w = int(rng.choice([1, 2, int(rng.integers(3, 130)), int(rng.integers(130, 1025)), int(rng.integers(1025, 3000))]))
    max_chunk = int(rng.integers(1, 700))
    sizes = [int(rng.integers(0, max_chunk + 1)) for _ in range(int(rng.integers(2, 9)))]
    total = sum(sizes)
    rows = _values(dtype, S * max(total, 1), 6000 + case).reshape(S, max(total, 1))
    st = mm.MaxMinStream(_tdt(dtype), S, w, max_chunk, device=DEV)
    exp = oracle.stream_pushes(rows, w, sizes)
    off = 0
    for k, c in enumerate(sizes):
        chunk_off = int(rng.integers(0, 3))
        ld = c + int(rng.integers(0, 4))
        buf = torch.zeros(chunk_off + S * max(ld, 1) + 8, dtype=_tdt(dtype), device=DEV)
        chunk = buf[chunk_off: chunk_off + S * ld].view(S, ld)[:, :c] if c > 0 else buf[:S].view(S, 1)[:, :0]
        if c > 0:
            chunk.copy_(torch.from_numpy(np.ascontiguousarray(rows[:, off: off + c])).to(DEV))
        ox, on, fv = st.push(chunk)
        ex, en = exp[k]
        if c > 0:
            e = ex.shape[1]  # windows the oracle's push completed
            _same(ox[:, c - e:].cpu().numpy(), ex, f"push {k} max c={c} w={w}")
            _same(on[:, c - e:].cpu().numpy(), en, f"push {k} min c={c} w={w}")
            assert fv == c - e or e == 0, (fv, c, e)
        off += c


# ------------------------------------------------------------------ 3-D boxes

@pytest.mark.parametrize("case", range(40))
def test_fuzz_3d(cuda_device, case):
    rng = np.random.default_rng(7000 + case)
    dtype = ALL[case % len(ALL)]
    depth, rows, cols = int(rng.integers(1, 24)), int(rng.integers(1, 70)), int(rng.integers(1, 150))
    wz, wy, wx = int(rng.integers(1, depth + 1)), int(rng.integers(1, min(rows, 20) + 1)), \
        int(rng.integers(1, min(cols, 30) + 1))
    vol = _values(dtype, depth * rows * cols, 7000 + case).reshape(depth, rows, cols)
    ld = cols + int(rng.integers(0, 5))
    t = torch.zeros(depth, rows, ld, dtype=_tdt(dtype), device=DEV)
    t[:, :, :cols] = torch.from_numpy(vol).to(DEV)
    mx, mn = mm.maxmin_filter_3d(t, wx, wy, wz, cols=cols)
    ex, en = oracle.separable_3d(vol, wx, wy, wz)
    what = f"{np.dtype(dtype).name} {depth}x{rows}x{cols} (ld {ld}) w={wx}x{wy}x{wz}"
    _same(mx.cpu().numpy(), ex, "max " + what)
    _same(mn.cpu().numpy(), en, "min " + what)
