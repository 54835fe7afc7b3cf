"""GPU parity at the bench's full sizes and on edge values.

* C4 in full: the 8 images of 16384^2 (the bench's launch configuration: every
  resident CTA of the packed-byte kernel walks ~28 tiles, so the cross-tile
  prefetch and the stage/ring reuse are compared element by element), image by
  image against the oracle's separable filter.
* C5 in full: all 2^30 - w + 1 windows for w in {7, 4096, 262144}, compared in
  chunks against the oracle's appendix listing (chunks filtered on host threads).
* C3 in full: all 65536 series of 4096 samples, w=129, in one batched call.
* Edge values (synth.edge_values): dtype extremes, +-inf, subnormals, long equal
  runs, through every kernel family: 1-D small / medium / large-window paths,
  batched rows, the 2-D packed-byte, separable and generic kernels, the arg
  filter, stream pushes, opening/closing and 3-D boxes.  Bit-exact: a flushed
  subnormal or a mis-ordered infinity changes output bits.
"""
import concurrent.futures as cf

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_cs_0610046_b200")


def bits(a):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
    a = np.ascontiguousarray(a)
    return a.view(np.dtype(f"u{a.dtype.itemsize}"))


def same(got, exp, what):
    g, e = bits(got), bits(exp)
    assert g.shape == e.shape, (what, g.shape, e.shape)
    if not np.array_equal(g, e):
        bad = np.flatnonzero((g != e).ravel())
        raise AssertionError(f"{what}: {bad.size} mismatches, first at flat index {bad[0]}")


DEV = torch.device("cuda:0")


# ------------------------------------------------------------------ full size

@pytest.mark.slow
def test_c4_full_size_every_image(cuda_device):
    """BASELINE config C4 in full: 8 x 16384^2 u8, 15x15, one call (the bench's)."""
    NI, R, C, w = synth.C4["batch"], synth.C4["rows"], synth.C4["cols"], synth.C4["w_row"]
    host = synth.c4()
    x = torch.from_numpy(host).to(DEV)
    Ro, Co = R - w + 1, C - w + 1
    ox = torch.empty(NI, Ro, C, dtype=torch.uint8, device=DEV)
    on = torch.empty_like(ox)
    mm.maxmin_filter_2d(x, w, w, out_max=ox[:, :, :Co], out_min=on[:, :, :Co])
    torch.cuda.synchronize()
    del x
    for b in range(NI):
        ex, en = oracle.separable_2d(host[b], w, w)
        same(ox[b, :, :Co], ex, f"C4 image {b} max")
        same(on[b, :, :Co], en, f"C4 image {b} min")


@pytest.mark.slow
def test_c3_full_size_every_row(cuda_device):
    """BASELINE config C3 in full: 65536 series x 4096, w=129, one batched call (the
    bench's), every row against the oracle (row blocks on host threads)."""
    B, n, w = synth.C3["batch"], synth.C3["n"], synth.C3["w"]
    host = synth.c3()
    x = torch.from_numpy(host).to(DEV)
    mx, mn = mm.maxmin_filter_batched(x, w)
    gx, gn = mx.cpu().numpy(), mn.cpu().numpy()
    del x, mx, mn
    blocks = [(r, min(r + 4096, B)) for r in range(0, B, 4096)]

    def one(b):
        return b, oracle.batched(host[b[0]:b[1]], w)

    with cf.ThreadPoolExecutor(max_workers=8) as pool:
        for (r0, r1), (ex, en) in pool.map(one, blocks):
            same(gx[r0:r1], ex, f"C3 rows {r0}..{r1} max")
            same(gn[r0:r1], en, f"C3 rows {r0}..{r1} min")


def _chunked_compare(a, w, gx, gn, chunk=1 << 25, threads=8):
    """Every window of a (length n) against oracle.appendix, in chunks of windows,
    each chunk filtered from its own slice on a host thread."""
    m = a.shape[0] - w + 1
    starts = list(range(0, m, chunk))

    def one(j0):
        k = min(chunk, m - j0)
        ex, en, _ = oracle.appendix(a[j0: j0 + k + w - 1], w)
        return j0, k, ex, en

    with cf.ThreadPoolExecutor(max_workers=threads) as ex_pool:
        for j0, k, ex, en in ex_pool.map(one, starts):
            same(gx[j0: j0 + k], ex, f"max w={w} chunk {j0}")
            same(gn[j0: j0 + k], en, f"min w={w} chunk {j0}")


@pytest.mark.slow
def test_c5_full_size_every_window(cuda_device):
    """BASELINE config C5 in full (n = 2^30): every window of every w."""
    n = synth.C5["n"]
    a = synth.c5(n)
    x = torch.from_numpy(a).to(DEV)
    for w in synth.C5["windows"]:
        ws = torch.empty(max(mm.maxmin_workspace_bytes(torch.float32, 1, n, w), 16), dtype=torch.uint8, device=DEV)
        mx, mn = mm.maxmin_filter_1d(x, w, workspace=ws)
        torch.cuda.synchronize()
        gx, gn = mx.cpu().numpy(), mn.cpu().numpy()
        del mx, mn, ws
        _chunked_compare(a, w, gx, gn)
        del gx, gn


# ---------------------------------------------------------------- edge values

EDGE_DTYPES = [np.uint8, np.int8, np.uint16, np.int16, np.uint32, np.int32, np.uint64, np.int64,
               np.float32, np.float64]
IDS = lambda d: np.dtype(d).name  # noqa: E731


@pytest.mark.parametrize("dtype", EDGE_DTYPES, ids=IDS)
def test_edge_values_1d_every_path(cuda_device, dtype):
    a = synth.edge_values(dtype, 120_001, seed=11)
    x = torch.from_numpy(a).to(DEV)
    for w in (2, 3, 16, 17, 129, 1024, 8193, 8194, 20_000):
        ws = torch.empty(max(mm.maxmin_workspace_bytes(x.dtype, 1, a.shape[0], w), 16), dtype=torch.uint8,
                         device=DEV)
        mx, mn = mm.maxmin_filter_1d(x, w, workspace=ws)
        ex, en, _ = oracle.appendix(a, w)
        same(mx, ex, f"{np.dtype(dtype).name} max w={w}")
        same(mn, en, f"{np.dtype(dtype).name} min w={w}")


@pytest.mark.parametrize("dtype", [np.uint8, np.int16, np.float32, np.float64], ids=IDS)
def test_edge_values_batched(cuda_device, dtype):
    rows, n = 9, 20_000
    a = synth.edge_values(dtype, rows * n, seed=12).reshape(rows, n)
    x = torch.from_numpy(a).to(DEV)
    for w in (5, 300, 9000):
        mx, mn = mm.maxmin_filter_batched(x, w)
        ex, en = oracle.batched(a, w)
        same(mx, ex, f"batched max w={w}")
        same(mn, en, f"batched min w={w}")


@pytest.mark.parametrize("dtype,wr,wc", [(np.uint8, 15, 15), (np.int8, 7, 7), (np.uint8, 6, 9),
                                         (np.float32, 5, 5), (np.float32, 15, 15), (np.float64, 7, 3),
                                         (np.int32, 33, 31), (np.uint16, 3, 17)], ids=str)
def test_edge_values_2d(cuda_device, dtype, wr, wc):
    """Packed-byte kernel (square <= 17 bytes), separable path, fused generic kernel."""
    b, R, C = 2, 300, 1040
    img = synth.edge_values(dtype, b * R * C, seed=13).reshape(b, R, C)
    x = torch.from_numpy(img).to(DEV)
    mx, mn = mm.maxmin_filter_2d(x, wr, wc)
    ex, en = oracle.separable_2d(img, wr, wc)
    same(mx, ex, f"2d max {wr}x{wc}")
    same(mn, en, f"2d min {wr}x{wc}")


@pytest.mark.parametrize("dtype", [np.uint8, np.int16, np.int32, np.float32], ids=IDS)
def test_edge_values_argfilter(cuda_device, dtype):
    """Long equal runs make the earliest-position rule (R17) bite."""
    a = synth.edge_values(dtype, 60_000, seed=14)
    x = torch.from_numpy(a).to(DEV)
    for w in (4, 100, 9000):
        mx, mn, ax, an = mm.maxmin_argfilter_1d(x, w)
        ex, en, eax, ean = oracle.arg_wedge(a, w)
        same(mx, ex, f"arg values max w={w}")
        same(mn, en, f"arg values min w={w}")
        same(ax, eax, f"argmax w={w}")
        same(an, ean, f"argmin w={w}")


@pytest.mark.parametrize("dtype", [np.uint8, np.int64, np.float32, np.float64], ids=IDS)
def test_edge_values_stream(cuda_device, dtype):
    S, c, w = 6, 300, 129
    rows = synth.edge_values(dtype, S * 4 * c, seed=15).reshape(S, 4 * c)
    st = mm.MaxMinStream(torch.from_numpy(rows[:1, :1]).dtype, S, w, c, device=DEV)
    got_x, got_n = [], []
    for p in range(4):
        ox, on, fv = st.push(torch.from_numpy(np.ascontiguousarray(rows[:, p * c:(p + 1) * c])).to(DEV))
        got_x.append(ox[:, fv:].cpu().numpy())
        got_n.append(on[:, fv:].cpu().numpy())
    ex, en = oracle.batched(rows, w)
    same(np.concatenate(got_x, axis=1), ex, "stream max")
    same(np.concatenate(got_n, axis=1), en, "stream min")


@pytest.mark.parametrize("dtype", [np.uint8, np.int32, np.float32, np.float64], ids=IDS)
def test_edge_values_morph(cuda_device, dtype):
    a = synth.edge_values(dtype, 4 * 5000, seed=16).reshape(4, 5000)
    x = torch.from_numpy(a).to(DEV)
    for w in (3, 129, 1025):
        op, cl = mm.maxmin_morph_batched(x, w)
        for r in range(4):
            eo, ec = oracle.morph(a[r], w)
            same(op[r], eo, f"open w={w} row {r}")
            same(cl[r], ec, f"close w={w} row {r}")
    img = synth.edge_values(dtype, 2 * 120 * 200, seed=17).reshape(2, 120, 200)
    op, cl = mm.maxmin_morph_2d(torch.from_numpy(img).to(DEV), 5, 7)
    eo, ec = oracle.morph_2d(img, 5, 7)
    same(op, eo, "open 2d")
    same(cl, ec, "close 2d")


@pytest.mark.parametrize("dtype", [np.uint8, np.float32], ids=IDS)
def test_edge_values_3d(cuda_device, dtype):
    vol = synth.edge_values(dtype, 20 * 64 * 96, seed=18).reshape(20, 64, 96)
    mx, mn = mm.maxmin_filter_3d(torch.from_numpy(vol).to(DEV), 5, 3, 4)
    ex, en = oracle.separable_3d(vol, 5, 3, 4)
    same(mx, ex, "3d max")
    same(mn, en, "3d min")


@pytest.mark.parametrize("dtype", [np.uint8, np.int8], ids=IDS)
@pytest.mark.parametrize("w", [2, 5, 15, 17])
def test_morph_2d_packed_framed_passes(cuda_device, dtype, w):
    """1-byte square-window opening/closing (three packed passes, the second and
    third reading through the tensor map's zero frame) on images spanning several
    512-column strips and 498-row bands, against the oracle's composition."""
    img = synth.c4(count=2, rows=1100, cols=1600, nrect=6)
    if dtype == np.int8:
        img = img.view(np.int8)
    op, cl = mm.maxmin_morph_2d(torch.from_numpy(img).to(DEV), w, w)
    eo, ec = oracle.morph_2d(img, w, w)
    same(op, eo, f"open {w}x{w}")
    same(cl, ec, f"close {w}x{w}")
