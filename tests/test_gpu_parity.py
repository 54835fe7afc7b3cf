"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit for
bit, on seeded inputs.  Sizes span several tiles and a ragged tail; every
kernel path (copy, small, medium, large), every dtype, batched rows and 2-D
images are covered, plus metamorphic checks that need no oracle at full size."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_cs_0610046_b200")


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.dtype(f"u{a.dtype.itemsize}"))


def assert_same(got, exp, what=""):
    got = got.cpu().numpy() if isinstance(got, torch.Tensor) else got
    assert got.shape == exp.shape, (what, got.shape, exp.shape)
    g, e = bits(got), bits(exp)
    if not np.array_equal(g, e):
        bad = np.flatnonzero((g != e).ravel())
        raise AssertionError(f"{what}: {bad.size} mismatches, first at {bad[0]}: "
                             f"got {got.ravel()[bad[0]]} expected {exp.ravel()[bad[0]]}")


def dev():
    return torch.device("cuda:0")


def run_1d(a, w):
    x = torch.from_numpy(a).to(dev())
    mx, mn = mm.maxmin_filter_1d(x, w)
    torch.cuda.synchronize()
    return mx, mn


# every path and the boundaries between them (E=16 for <=4-byte types)
W_1D = [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 18, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256,
        257, 511, 512, 513, 1023, 1024, 1025, 2047, 2049, 4095, 4096, 4097, 4098, 8191, 8192, 8193,
        8194, 8195, 12289, 20000, 65536]


@pytest.mark.parametrize("w", W_1D)
def test_1d_f32_all_paths(cuda_device, w):
    n = 100_003  # several tiles of 4096 + ragged tail
    a = synth.c2(n)
    mx, mn = run_1d(a, w)
    ex, en, _ = oracle.appendix(a, w)
    assert_same(mx, ex, f"max w={w}")
    assert_same(mn, en, f"min w={w}")


@pytest.mark.parametrize("n_minus_w", [0, 1, 2, 15, 4095, 4096, 4097])
@pytest.mark.parametrize("w", [1, 3, 16, 17, 300, 8193, 9000])
def test_1d_short_inputs(cuda_device, w, n_minus_w):
    n = w + n_minus_w
    a = synth.random_values(np.float32, n, seed=w * 7 + n_minus_w)
    mx, mn = run_1d(a, w)
    ex, en, _ = oracle.brute_1d(a, w) if n * w < 5e7 else oracle.appendix(a, w)
    assert_same(mx, ex, f"max n={n} w={w}")
    assert_same(mn, en, f"min n={n} w={w}")


DTYPES = [np.uint8, np.int8, np.uint16, np.int16, np.uint32, np.int32, np.uint64, np.int64,
          np.float32, np.float64]


@pytest.mark.parametrize("dtype", DTYPES, ids=lambda d: np.dtype(d).name)
@pytest.mark.parametrize("alphabet", [None, 5])
def test_1d_every_dtype(cuda_device, dtype, alphabet):
    n = 50_001
    for k, w in enumerate([2, 3, 8, 9, 16, 17, 100, 1000, 5000, 8193, 10_000]):
        a = synth.random_values(dtype, n, seed=1000 + k, alphabet=alphabet)
        mx, mn = run_1d(a, w)
        ex, en, _ = oracle.appendix(a, w)
        assert_same(mx, ex, f"{np.dtype(dtype).name} max w={w}")
        assert_same(mn, en, f"{np.dtype(dtype).name} min w={w}")


def test_1d_single_output(cuda_device):
    a = synth.c2(70_000)
    x = torch.from_numpy(a).to(dev())
    for w in (3, 100, 9000):
        ex, en, _ = oracle.appendix(a, w)
        mx, mn = mm.maxmin_filter_1d(x, w, want_min=False)
        assert mn is None
        assert_same(mx, ex)
        mx, mn = mm.maxmin_filter_1d(x, w, want_max=False)
        assert mx is None
        assert_same(mn, en)


def test_c1_config(cuda_device):
    """BASELINE config C1: f64 i.i.d. U[0,1), n=100000, w=16, against brute force."""
    a = synth.c1()
    mx, mn = run_1d(a, 16)
    ex, en, st = oracle.brute_1d(a, 16)
    assert_same(mx, ex)
    assert_same(mn, en)


@pytest.mark.parametrize("w", [2, 17, 129, 4000, 9000])
def test_batched_rows(cuda_device, w):
    rows, n, ld = 37, 10_000, 10_016
    base = synth.c3(rows=rows, length=n, ld=ld)
    x = torch.from_numpy(base).to(dev())
    mx, mn = mm.maxmin_filter_batched(x, w, n=n)
    torch.cuda.synchronize()
    ex, en = oracle.batched(base, w, n=n)
    assert_same(mx, ex, f"batched max w={w}")
    assert_same(mn, en, f"batched min w={w}")


@pytest.mark.parametrize("dtype", [np.uint8, np.int8, np.float32, np.float64],
                         ids=lambda d: np.dtype(d).name)
def test_large_window_repeated(cuda_device, dtype):
    """The look-back kernel's ticket ring, many rows and many launches: each row
    starts with q publishing-only tickets, so ordering bugs between the stage
    warp and the publish step show up as sporadic mismatches or faults."""
    rows, n = 24, 40_000
    a = synth.random_values(dtype, rows * n, seed=4242).reshape(rows, n)
    x = torch.from_numpy(a).to(dev())
    for w in (8194, 10_000, 17_000, 39_999):
        ex, en = oracle.batched(a, w)
        for _ in range(10):
            mx, mn = mm.maxmin_filter_batched(x, w)
            torch.cuda.synchronize()
            assert_same(mx, ex, f"max w={w}")
            assert_same(mn, en, f"min w={w}")


@pytest.mark.parametrize("w", [8193 + 512, 9000, 9600, 9985])
def test_large_window_publish_only_rows(cuda_device, w):
    """Rows only a few tiles longer than the window (n=10000, q = 17..19): most of
    every row's groups are publish-only for warp 0 (its tile lies before the row's
    first window), so warp 0 takes no waits of its own there.  Every live job
    waits for its table stage (k1d_lw.cuh pipeline), which bounds how far warp 0
    can run ahead of siblings stuck on gap polls; without it a longer ticket
    lead (-DMM_LW_TL3=9) faulted here.  Repeated launches, 300 rows."""
    rows, n = 300, 10_000
    a = synth.random_values(np.float32, rows * n, seed=777).reshape(rows, n)
    x = torch.from_numpy(a).to(dev())
    ex, en = oracle.batched(a, w)
    for _ in range(8):
        mx, mn = mm.maxmin_filter_batched(x, w)
        torch.cuda.synchronize()
        assert_same(mx, ex, f"max w={w}")
        assert_same(mn, en, f"min w={w}")


def test_c3_shape_sample(cuda_device):
    """C3 layout [65536][4096] f32, w=129; parity on a 2048-row slice (full size in bench)."""
    rows = 2048
    b = synth.c3(rows=rows, row0=12345)
    x = torch.from_numpy(b).to(dev())
    mx, mn = mm.maxmin_filter_batched(x, 129)
    ex, en = oracle.batched(b, 129)
    assert_same(mx, ex)
    assert_same(mn, en)


@pytest.mark.parametrize("wr,wc", [(1, 1), (1, 7), (7, 1), (2, 2), (3, 5), (15, 15), (16, 16),
                                   (17, 9), (33, 31)])
def test_2d_u8(cuda_device, wr, wc):
    img = synth.c4(count=3, rows=301, cols=517, nrect=10)
    x = torch.from_numpy(img).to(dev())
    mx, mn = mm.maxmin_filter_2d(x, wr, wc)
    ex, en = oracle.separable_2d(img, wr, wc)
    assert_same(mx, ex, f"2d max {wr}x{wc}")
    assert_same(mn, en, f"2d min {wr}x{wc}")


@pytest.mark.parametrize("dtype", DTYPES, ids=lambda d: np.dtype(d).name)
def test_2d_every_dtype(cuda_device, dtype):
    a = synth.random_values(dtype, 2 * 90 * 160, seed=77).reshape(2, 90, 160)
    x = torch.from_numpy(a).to(dev())
    for wr, wc in ((3, 4), (15, 15), (9, 1)):
        mx, mn = mm.maxmin_filter_2d(x, wr, wc)
        ex, en = oracle.brute_2d(a, wr, wc)
        assert_same(mx, ex, f"2d max {wr}x{wc}")
        assert_same(mn, en, f"2d min {wr}x{wc}")


def test_2d_strided_output(cuda_device):
    """C4 convention: outputs with a padded row pitch (out_ld = cols)."""
    img = synth.c4(count=2, rows=256, cols=512, nrect=6)
    x = torch.from_numpy(img).to(dev())
    R, C = 256 - 14, 512 - 14
    ox = torch.zeros(2, R, 512, dtype=torch.uint8, device=dev())
    on = torch.zeros(2, R, 512, dtype=torch.uint8, device=dev())
    mm.maxmin_filter_2d(x, 15, 15, out_max=ox[:, :, :C], out_min=on[:, :, :C])
    ex, en = oracle.separable_2d(img, 15, 15)
    assert_same(ox[:, :, :C].contiguous(), ex)
    assert_same(on[:, :, :C].contiguous(), en)
    assert int(ox[:, :, C:].abs().sum()) == 0  # padding untouched


# ------------------------------------------------------------ metamorphic ---

@pytest.mark.parametrize("w", [3, 32, 1024, 65536])
def test_shift_invariance(cuda_device, w):
    """F(a[s:]) = F(a)[s:]: moves every tile/halo seam (no oracle needed)."""
    a = synth.c2(1 << 22)
    x = torch.from_numpy(a).to(dev())
    mx, mn = mm.maxmin_filter_1d(x, w)
    for s in (4, 1000, 4096 * 3 + 8):
        sx, sn = mm.maxmin_filter_1d(x[s:].contiguous(), w)
        assert torch.equal(sx, mx[s:]) and torch.equal(sn, mn[s:]), s


def test_dilation_semigroup(cuda_device):
    """max_{w1} o max_{w2} = max_{w1+w2-1}: checks the large path against compositions."""
    a = synth.c2(1 << 21)
    x = torch.from_numpy(a).to(dev())
    for w1, w2 in ((4097, 8192), (30000, 35537), (3, 65534)):
        m1, n1 = mm.maxmin_filter_1d(x, w1)
        m12, _ = mm.maxmin_filter_1d(m1, w2, want_min=False)
        _, n12 = mm.maxmin_filter_1d(n1, w2, want_max=False)
        mw, nw = mm.maxmin_filter_1d(x, w1 + w2 - 1)
        assert torch.equal(m12, mw) and torch.equal(n12, nw), (w1, w2)


def test_u8_complement(cuda_device):
    a = synth.uniform_u8(5, 0, 300_000)
    x = torch.from_numpy(a).to(dev())
    for w in (3, 40, 10_000):
        mx, mn = mm.maxmin_filter_1d(x, w)
        cx, cn = mm.maxmin_filter_1d(255 - x, w)
        assert torch.equal(mn, 255 - cx) and torch.equal(mx, 255 - cn)


# ------------------------------------------------------------- full size ----

def test_c2_full_size(cuda_device):
    """BASELINE config C2 at full size (n = 2^28) for every window, vs the oracle."""
    n = 1 << 28
    a = synth.c2(n)
    x = torch.from_numpy(a).to(dev())
    for w in (3, 32, 1024, 65536):
        mx, mn = mm.maxmin_filter_1d(x, w)
        ex, en, _ = oracle.appendix(a, w)
        assert_same(mx, ex, f"C2 max w={w}")
        del ex
        assert_same(mn, en, f"C2 min w={w}")
        del mx, mn, en


def test_c5_full_size_sampled(cuda_device):
    """BASELINE config C5 (n = 2^30): windows around tile seams and random spots,
    each recomputed by the oracle on the slice that contains it."""
    n = 1 << 30
    a = synth.c5(n)
    x = torch.from_numpy(a).to(dev())
    rng = np.random.default_rng(5)
    for w in (7, 4096, 262144):
        mx, mn = mm.maxmin_filter_1d(x, w)
        m = n - w + 1
        starts = [0, 4096 - 3, 4096 * 1000 - 1, m - 5000] + list(rng.integers(0, m - 5000, 6))
        for j0 in starts:
            j0 = int(j0)
            k = 4096 + 37
            sl = a[j0: j0 + k + w - 1]
            ex, en, _ = oracle.appendix(sl, w)
            assert_same(mx[j0: j0 + ex.shape[0]], ex, f"C5 max w={w} j0={j0}")
            assert_same(mn[j0: j0 + en.shape[0]], en, f"C5 min w={w} j0={j0}")
        del mx, mn
    del x


def test_host_pipeline(cuda_device):
    a = synth.c2(3_000_017)
    for w in (3, 1024, 70000):
        ex, en, _ = oracle.appendix(a, w)
        x = torch.from_numpy(a).pin_memory()
        ox = torch.empty(ex.shape[0], dtype=torch.float32).pin_memory()
        on = torch.empty(ex.shape[0], dtype=torch.float32).pin_memory()
        chunk = 1 << 20
        ws = torch.empty(mm.maxmin_host_workspace_bytes(torch.float32, a.shape[0], w, chunk),
                         dtype=torch.uint8, device=dev())
        mm.maxmin_filter_1d_host(x, w, ox, on, ws, chunk=chunk)
        assert_same(ox.numpy(), ex)
        assert_same(on.numpy(), en)


def test_device_errors(cuda_device):
    x = torch.from_numpy(synth.c2(100_000)).to(dev())
    with pytest.raises(mm.MaxMinError) as e:
        mm.maxmin_filter_1d(x, 70_000, workspace=torch.empty(16, dtype=torch.uint8, device=dev()))
    assert e.value.status == 8
    L = mm._lib.lib()
    host = torch.zeros(1000).pin_memory()
    out = torch.empty(998, device=dev())
    rc = L.maxmin_filter_1d(8, host.data_ptr(), 1000, 3, out.data_ptr(), None, None, 0, None)
    assert rc == 11  # host pointer passed to the device API


# ------------------------------------------------- packed 1-byte 2-D path ---
# k2d_byte takes square windows 2..17 when rows/pitches are 16-B multiples;
# shapes below span several 1024-column strips, ragged right edges, short
# images and CTA row ranges that straddle images.
BYTE_W = [2, 3, 4, 5, 7, 9, 11, 13, 15, 16, 17]


@pytest.mark.parametrize("w", BYTE_W)
@pytest.mark.parametrize("dtype", [np.uint8, np.int8], ids=lambda d: np.dtype(d).name)
def test_2d_byte_fast_path(cuda_device, w, dtype):
    img = synth.c4(count=3, rows=203, cols=2096, nrect=12)
    if dtype == np.int8:
        img = img.view(np.int8)
    x = torch.from_numpy(img).to(dev())
    mx, mn = mm.maxmin_filter_2d(x, w, w)
    ex, en = oracle.separable_2d(img, w, w)
    assert_same(mx, ex, f"2d max {w}x{w}")
    assert_same(mn, en, f"2d min {w}x{w}")


@pytest.mark.parametrize("shape", [(1, 15, 16), (2, 15, 1040), (5, 40, 1024), (1, 700, 3088),
                                   (9, 17, 1056), (2, 1000, 48)])
def test_2d_byte_shapes(cuda_device, shape):
    b, r, c = shape
    img = synth.c4(count=b, rows=r, cols=c, nrect=4)
    x = torch.from_numpy(img).to(dev())
    for w in (15, 3):
        if w > r:
            continue
        mx, mn = mm.maxmin_filter_2d(x, w, w)
        ex, en = oracle.separable_2d(img, w, w)
        assert_same(mx, ex, f"2d max {shape} w={w}")
        assert_same(mn, en, f"2d min {shape} w={w}")


def test_2d_byte_strided_single_output(cuda_device):
    """C4 output convention (out_ld = cols, 16-B rows) and one output only."""
    img = synth.c4(count=2, rows=300, cols=2048, nrect=6)
    x = torch.from_numpy(img).to(dev())
    R, C = 300 - 14, 2048 - 14
    ox = torch.zeros(2, R, 2048, dtype=torch.uint8, device=dev())
    on = torch.zeros(2, R, 2048, dtype=torch.uint8, device=dev())
    ex, en = oracle.separable_2d(img, 15, 15)
    mm.maxmin_filter_2d(x, 15, 15, out_max=ox[:, :, :C], want_min=False)
    mm.maxmin_filter_2d(x, 15, 15, out_min=on[:, :, :C], want_max=False)
    assert_same(ox[:, :, :C].contiguous(), ex)
    assert_same(on[:, :, :C].contiguous(), en)
    assert int(ox[:, :, C:].sum()) == 0 and int(on[:, :, C:].sum()) == 0


# ------------------------------------------------------- N1: arg filter ----
ARG_DTYPES = [np.uint8, np.int8, np.uint16, np.int16, np.uint32, np.int32, np.float32]


@pytest.mark.parametrize("dtype", ARG_DTYPES, ids=lambda d: np.dtype(d).name)
def test_argfilter_every_dtype(cuda_device, dtype):
    """Values and earliest positions of max/min vs the definition, with ties
    (small alphabets) and every kernel path of the key filters."""
    n = 20_003
    for k, w in enumerate([1, 2, 3, 7, 8, 9, 16, 17, 100, 129, 1000, 1025, 1026, 5000, 9000]):
        a = synth.random_values(dtype, n, seed=2000 + k, alphabet=(4 if k % 2 else None))
        x = torch.from_numpy(a).to(dev())
        mx, mn, ax, an = mm.maxmin_argfilter_1d(x, w)
        ex, en, eax, ean = oracle.arg_wedge(a, w)
        assert_same(mx, ex, f"{np.dtype(dtype).name} max w={w}")
        assert_same(mn, en, f"{np.dtype(dtype).name} min w={w}")
        assert_same(ax, eax, f"{np.dtype(dtype).name} argmax w={w}")
        assert_same(an, ean, f"{np.dtype(dtype).name} argmin w={w}")


def test_argfilter_brute_and_batched(cuda_device):
    a = synth.random_values(np.float32, 3 * 2500, seed=31, alphabet=6).reshape(3, 2500)
    x = torch.from_numpy(a).to(dev())
    for w in (5, 77, 2500):
        mx, mn, ax, an = mm.maxmin_argfilter_batched(x, w)
        for r in range(3):
            ex, en, eax, ean = oracle.arg_brute(a[r], w)
            assert_same(ax[r], eax, f"row {r} argmax w={w}")
            assert_same(an[r], ean, f"row {r} argmin w={w}")
            assert_same(mx[r], ex)
            assert_same(mn[r], en)
    # one side only, positions only
    _, _, ax, an = mm.maxmin_argfilter_batched(x, 77, want_min=False, values=False)
    assert an is None
    assert_same(ax[1], oracle.arg_brute(a[1], 77)[2])


def test_argfilter_unaligned_rows_and_outputs(cuda_device):
    """Odd input pitch and odd output pitch through the C ABI: the fused kernel's
    element-wise staging and scalar stores."""
    import ctypes

    batch, n, ld, w = 5, 3001, 3003, 129
    a = synth.random_values(np.int16, batch * ld, seed=77, alphabet=5).reshape(batch, ld)
    x = torch.from_numpy(a).to(dev())
    m = n - w + 1
    out_ld = m + 1
    ox = torch.empty(batch * out_ld + 1, dtype=torch.int16, device=dev())[1:]  # 2-B aligned only
    on = torch.empty_like(ox)
    ax = torch.empty(batch * out_ld, dtype=torch.int64, device=dev())
    an = torch.empty_like(ax)
    L = mm._lib.lib()
    vp = ctypes.c_void_p
    need = mm.maxmin_argfilter_workspace_bytes(torch.int16, batch, n, w)
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device=dev())
    mm._lib.check(L.maxmin_argfilter_batched(mm.dtype_code(torch.int16), vp(x.data_ptr()), batch, n, ld, w,
                                             vp(ox.data_ptr()), vp(on.data_ptr()), vp(ax.data_ptr()),
                                             vp(an.data_ptr()), out_ld, vp(ws.data_ptr()), ws.numel(),
                                             vp(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    for r in range(batch):
        ex, en, eax, ean = oracle.arg_brute(a[r, :n], w)
        sl = slice(r * out_ld, r * out_ld + m)
        assert_same(ox[sl], ex, f"row {r} max")
        assert_same(on[sl], en, f"row {r} min")
        assert_same(ax[sl], eax, f"row {r} argmax")
        assert_same(an[sl], ean, f"row {r} argmin")


@pytest.mark.parametrize("w", [5, 129, 1024])
def test_single_row_pitch_is_free(cuda_device, w):
    """One row through the C ABI with the natural pitches (in_ld = n, out_ld = m, both
    odd): a pitch never enters an address when batch == 1, so the vector paths run
    (the bench's N1 call) and the results match the oracle."""
    import ctypes

    n = 40_001
    m = n - w + 1
    a = synth.random_values(np.float32, n, seed=90 + w, alphabet=7)
    x = torch.from_numpy(a).to(dev())
    L = mm._lib.lib()
    vp = ctypes.c_void_p
    s = vp(torch.cuda.current_stream().cuda_stream)
    code = mm.dtype_code(torch.float32)
    ox, on = torch.empty(m, device=dev()), torch.empty(m, device=dev())
    ax = torch.empty(m, dtype=torch.int64, device=dev())
    an = torch.empty_like(ax)
    need = mm.maxmin_argfilter_workspace_bytes(torch.float32, 1, n, w)
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device=dev())
    mm._lib.check(L.maxmin_argfilter_batched(code, vp(x.data_ptr()), 1, n, n, w, vp(ox.data_ptr()),
                                             vp(on.data_ptr()), vp(ax.data_ptr()), vp(an.data_ptr()), m,
                                             vp(ws.data_ptr()), ws.numel(), s))
    op, cl = torch.empty(n, device=dev()), torch.empty(n, device=dev())
    mm._lib.check(L.maxmin_morph_batched(code, vp(x.data_ptr()), 1, n, n, w, vp(op.data_ptr()),
                                         vp(cl.data_ptr()), n, s))
    torch.cuda.synchronize()
    ex, en, eax, ean = oracle.arg_wedge(a, w)
    assert_same(ox, ex, "arg values max")
    assert_same(on, en, "arg values min")
    assert_same(ax, eax, "argmax")
    assert_same(an, ean, "argmin")
    eo, ec = oracle.morph(a, w)
    assert_same(op, eo, "opening")
    assert_same(cl, ec, "closing")


def test_argfilter_c2_full_size(cuda_device):
    """C2's array (n = 2^28) at w = 1024: positions vs the wedge oracle."""
    a = synth.c2(1 << 28)
    x = torch.from_numpy(a).to(dev())
    mx, mn, ax, an = mm.maxmin_argfilter_1d(x, 1024)
    ex, en, eax, ean = oracle.arg_wedge(a, 1024)
    assert_same(ax, eax, "argmax")
    assert_same(an, ean, "argmin")
    assert_same(mx, ex)
    assert_same(mn, en)


# ------------------------------------------------------------ N3: LB_Keogh ---
def _keogh_close(got, exp):
    got = got.cpu().numpy() if isinstance(got, torch.Tensor) else got
    err = np.abs(got - exp) / np.maximum(1.0, np.abs(exp))
    assert np.all(err <= 1e-12), (float(err.max()), int(err.argmax()))


@pytest.mark.parametrize("r", [0, 1, 3, 7, 8, 40, 64, 300, 1000, 4096])
def test_keogh_radii(cuda_device, r):
    """Small (w <= 16), medium and clipped-only (2r+1 > n) paths, ragged rows."""
    rows, n, ld = 19, 3001, 3004
    c = synth.c3(rows=rows, length=n, ld=ld)
    q = synth.c3(rows=1, length=n, row0=777)[0]
    x = torch.from_numpy(c).to(dev())
    qd = torch.from_numpy(q).to(dev())
    lb = mm.maxmin_lb_keogh_batched(x, qd, r, n=n)
    _keogh_close(lb, oracle.keogh(c[:, :n], q, r))


def test_keogh_short_rows_and_identity(cuda_device):
    for n in (1, 2, 5, 31, 33, 129):
        ld = (n + 3) // 4 * 4  # 16-byte row pitch (the C ABI's rule)
        c = synth.random_values(np.float32, 8 * ld, seed=n).reshape(8, ld)
        q = synth.random_values(np.float32, n, seed=1000 + n)
        for r in (0, 1, 2, 16, 64, 200):
            lb = mm.maxmin_lb_keogh_batched(torch.from_numpy(c).to(dev()), torch.from_numpy(q).to(dev()), r, n=n)
            _keogh_close(lb, oracle.keogh(c[:, :n], q, r))
    c = synth.c3(rows=4, length=512)
    lb = mm.maxmin_lb_keogh_batched(torch.from_numpy(c).to(dev()), torch.from_numpy(c[2].copy()).to(dev()), 64)
    assert float(lb[2]) == 0.0


def test_keogh_c3_shape_sample(cuda_device):
    """C3's layout (4096-sample series, w = 129 -> r = 64) on a 4096-row slice."""
    c = synth.c3(rows=4096, row0=4321)
    q = synth.c3(rows=1, row0=65536)[0]
    lb = mm.maxmin_lb_keogh_batched(torch.from_numpy(c).to(dev()), torch.from_numpy(q).to(dev()), 64)
    _keogh_close(lb, oracle.keogh(c, q, 64))


# ------------------------------------------------------------- N2: streams
def _stream_check(dtype, streams, w, sizes, max_chunk, seed, pitch=None):
    N = int(sum(sizes))
    rows = np.stack([synth.random_values(np.dtype(dtype), max(N, 1), seed=seed, stream=s)[:N]
                     for s in range(streams)]) if streams else np.empty((0, N), dtype)
    exp = oracle.stream_pushes(rows, w, sizes)
    st = mm.MaxMinStream(torch.from_numpy(np.empty(0, dtype)).dtype, streams, w, max_chunk, device=dev())
    x = torch.from_numpy(rows).to(dev())
    off = 0
    for p, c in enumerate(sizes):
        if pitch is None:
            ch = x[:, off:off + c].contiguous()
        else:  # chunk rows at an odd pitch: element-wise staging
            ch = torch.empty(streams, c + pitch, dtype=x.dtype, device=dev())[:, :c]
            ch.copy_(x[:, off:off + c])
        mx, mn, fv = st.push(ch)
        torch.cuda.synchronize()
        ex, en = exp[p]
        e = ex.shape[1] if streams else max(0, min(c, off + c - w + 1))
        assert fv == c - e, (p, c, fv, e)
        if streams and e:
            assert_same(mx[:, fv:], ex, f"max push {p} (c={c})")
            assert_same(mn[:, fv:], en, f"min push {p} (c={c})")
        off += c
    assert st.seen == N


@pytest.mark.parametrize("w", [1, 2, 3, 16, 17, 18, 33, 129, 200, 513, 600, 1000, 1025, 1026, 4097, 9000])
def test_stream_pushes_f32(cuda_device, w):
    rng = np.random.default_rng(w)
    max_chunk = 1500
    sizes = [0, 1, 2, min(w // 2, max_chunk), max_chunk, 3, w + 5 if w + 5 <= max_chunk else 700] + \
        rng.integers(0, max_chunk + 1, size=8).tolist()
    _stream_check(np.float32, 37, w, sizes, max_chunk, seed=w)


@pytest.mark.parametrize("dtype", DTYPES, ids=lambda d: np.dtype(d).name)
def test_stream_every_dtype(cuda_device, dtype):
    for w in (5, 17, 300, 1025, 9000):
        sizes = [100, 4000, 7, 2999, 4096, 1]
        _stream_check(dtype, 9, w, sizes, 4096, seed=w + 1)


def test_stream_odd_chunk_pitch(cuda_device):
    _stream_check(np.float32, 64, 129, [256] * 6 + [13, 255], 256, seed=5, pitch=1)
    _stream_check(np.uint8, 64, 40, [256] * 3 + [13, 255], 256, seed=6, pitch=3)


@pytest.mark.parametrize("w", [200, 600, 1025])
def test_stream_many_segments_per_warp(cuda_device, w):
    """Enough streams that every warp of the persistent grid runs many segments (its
    staging ring and aggregate slots are reused) with a non-empty gap (w-1 not a block)."""
    streams, c = 20000, 300
    rows = synth.c3(rows=streams, length=4 * c)
    st = mm.MaxMinStream(torch.float32, streams, w, c, device=dev())
    x = torch.from_numpy(rows).to(dev())
    exp = oracle.stream_pushes(rows[:64], w, [c] * 4)
    k = np.random.default_rng(w).choice(streams, 64, replace=False)
    expk = oracle.stream_pushes(rows[k], w, [c] * 4)
    for p in range(4):
        mx, mn, fv = st.push(x[:, p * c:(p + 1) * c].contiguous())
        torch.cuda.synchronize()
        assert_same(mx[:64, fv:], exp[p][0], f"max push {p}")
        assert_same(mn[:64, fv:], exp[p][1], f"min push {p}")
        assert_same(mx[k, fv:], expk[p][0], f"max push {p} sampled")
        assert_same(mn[k, fv:], expk[p][1], f"min push {p} sampled")


def test_stream_c3_full_size(cuda_device):
    """C3's 65 536 series as streams, 16 pushes of 256 samples, w=129 (the N2 bench
    workload): every window against the oracle's batch filter on the whole rows
    (streaming = batch) -- all rows, all windows."""
    rows = synth.c3()
    w, c = 129, 256
    st = mm.MaxMinStream(torch.float32, rows.shape[0], w, c, device=dev())
    x = torch.from_numpy(rows).to(dev())
    gx = torch.empty(rows.shape[0], rows.shape[1] - w + 1, dtype=torch.float32)
    gn = torch.empty_like(gx)
    k = 0
    for p in range(rows.shape[1] // c):
        mx, mn, fv = st.push(x[:, p * c:(p + 1) * c].contiguous())
        e = c - fv
        gx[:, k:k + e] = mx[:, fv:].cpu()
        gn[:, k:k + e] = mn[:, fv:].cpu()
        k += e
    assert k == rows.shape[1] - w + 1
    ex, en = oracle.batched(rows, w)
    assert_same(gx, ex, "C3 stream max")
    assert_same(gn, en, "C3 stream min")


# ------------------------------------------------------------- N4: morphology
MORPH_W = [1, 2, 3, 5, 8, 15, 16, 17, 18, 31, 33, 64, 129, 200, 513, 600, 1025, 1026, 3000, 8193]


@pytest.mark.parametrize("w", MORPH_W)
def test_morph_f32_windows(cuda_device, w):
    n = 9_001  # several segments of 512 + a ragged tail
    rows = np.stack([synth.c2(n, stream=s) for s in range(3)])
    x = torch.from_numpy(rows).to(dev())
    op, cl = mm.maxmin_morph_batched(x, w)
    torch.cuda.synchronize()
    for b in range(3):
        eo, ec = oracle.morph(rows[b], w)
        assert_same(op[b], eo, f"open row {b} w={w}")
        assert_same(cl[b], ec, f"close row {b} w={w}")


@pytest.mark.parametrize("dtype", DTYPES, ids=lambda d: np.dtype(d).name)
def test_morph_every_dtype(cuda_device, dtype):
    for w in (3, 8, 9, 16, 17, 100, 1000):
        n = 5000
        a = synth.random_values(np.dtype(dtype), 2 * n, seed=w)
        rows = a.reshape(2, n)
        x = torch.from_numpy(rows).to(dev())
        op, cl = mm.maxmin_morph_batched(x, w)
        torch.cuda.synchronize()
        for b in range(2):
            eo, ec = oracle.morph(rows[b], w)
            assert_same(op[b], eo, f"open {np.dtype(dtype).name} w={w}")
            assert_same(cl[b], ec, f"close {np.dtype(dtype).name} w={w}")


@pytest.mark.parametrize("n_minus_w", [0, 1, 2, 100])
@pytest.mark.parametrize("w", [1, 4, 17, 300])
def test_morph_short_rows_and_brute(cuda_device, w, n_minus_w):
    n = w + n_minus_w
    a = synth.random_values(np.float32, n, seed=n)
    x = torch.from_numpy(a).to(dev())
    op, cl = mm.maxmin_morph_1d(x, w)
    torch.cuda.synchronize()
    eo, ec = oracle.morph(a, w, brute=n * w * w < 3e7)
    assert_same(op, eo, "open")
    assert_same(cl, ec, "close")


def test_morph_strided_rows_and_one_output(cuda_device):
    rows = synth.c3(rows=50, length=1000, ld=1003)  # odd input pitch: element-wise staging
    x = torch.from_numpy(rows).to(dev())
    op, _ = mm.maxmin_morph_batched(x, 129, n=1000, want_close=False)
    _, cl = mm.maxmin_morph_batched(x, 129, n=1000, want_open=False)
    torch.cuda.synchronize()
    for b in (0, 17, 49):
        eo, ec = oracle.morph(rows[b, :1000], 129)
        assert_same(op[b], eo, "open")
        assert_same(cl[b], ec, "close")


def test_morph_c3_full_size_sampled(cuda_device):
    """C3's 65 536 x 4096 series, w=129 (the N4 bench workload): 300 sampled rows."""
    rows = synth.c3()
    x = torch.from_numpy(rows).to(dev())
    op, cl = mm.maxmin_morph_batched(x, 129)
    torch.cuda.synchronize()
    for b in np.random.default_rng(2).choice(rows.shape[0], 300, replace=False):
        eo, ec = oracle.morph(rows[b], 129)
        assert_same(op[b], eo, f"open row {b}")
        assert_same(cl[b], ec, f"close row {b}")


@pytest.mark.parametrize("wr,wc", [(1, 1), (3, 3), (5, 2), (1, 7), (15, 15), (16, 16), (4, 9)])
@pytest.mark.parametrize("dtype", [np.uint8, np.float32, np.int64], ids=lambda d: np.dtype(d).name)
def test_morph_2d(cuda_device, wr, wc, dtype):
    a = synth.random_values(np.dtype(dtype), 2 * 70 * 90, seed=wr * 31 + wc).reshape(2, 70, 90)
    x = torch.from_numpy(a).to(dev())
    op, cl = mm.maxmin_morph_2d(x, wr, wc)
    torch.cuda.synchronize()
    eo, ec = oracle.morph_2d(a, wr, wc)
    assert_same(op, eo, "open 2d")
    assert_same(cl, ec, "close 2d")


# ------------------------------------------------ NEXT rows: API corner cases
def test_stream_single_output_and_reuse(cuda_device):
    """One output array per push (max only / min only), preallocated outputs reused."""
    rows = synth.c3(rows=33, length=600)
    w, c = 40, 150
    x = torch.from_numpy(rows).to(dev())
    exp = oracle.stream_pushes(rows, w, [c] * 4)
    sx = mm.MaxMinStream(torch.float32, 33, w, c, device=dev())
    sn = mm.MaxMinStream(torch.float32, 33, w, c, device=dev())
    ox = torch.empty(33, 152, dtype=torch.float32, device=dev())[:, :c]
    on = torch.empty(33, 152, dtype=torch.float32, device=dev())[:, :c]
    for p in range(4):
        ch = x[:, p * c:(p + 1) * c].contiguous()
        mx, none1, fv = sx.push(ch, out_max=ox, want_min=False)
        none2, mn, fv2 = sn.push(ch, out_min=on, want_max=False)
        torch.cuda.synchronize()
        assert none1 is None and none2 is None and fv == fv2
        assert_same(mx[:, fv:], exp[p][0], f"max push {p}")
        assert_same(mn[:, fv:], exp[p][1], f"min push {p}")


def test_morph_2d_strided_input_single_output(cuda_device):
    a = synth.random_values(np.float32, 3 * 50 * 70, seed=12).reshape(3, 50, 70)
    x = torch.from_numpy(a).to(dev())
    op, cl = mm.maxmin_morph_2d(x, 5, 3, cols=61, want_close=False)  # the first 61 columns of each row
    torch.cuda.synchronize()
    assert cl is None
    eo, _ = oracle.morph_2d(np.ascontiguousarray(a[:, :, :61]), 5, 3)
    assert_same(op, eo, "open 2d strided")


def test_keogh_rows_shorter_than_pitch(cuda_device):
    c = synth.c3(rows=20, length=1000, ld=1004)
    q = synth.c3(rows=1, row0=99, length=1000)[0]
    lb = mm.maxmin_lb_keogh_batched(torch.from_numpy(c).to(dev()), torch.from_numpy(q).to(dev()), 30, n=1000)
    ref = oracle.keogh(np.ascontiguousarray(c[:, :1000]), q, 30)
    _keogh_close(lb, ref)


# ------------------------------------------------------------ N4: 3-D boxes
@pytest.mark.parametrize("dtype", [np.uint8, np.float32, np.int64, np.float64], ids=lambda d: np.dtype(d).name)
@pytest.mark.parametrize("wx,wy,wz", [(1, 1, 1), (3, 3, 3), (5, 2, 4), (15, 15, 5), (1, 7, 9), (16, 16, 2)])
def test_3d_boxes(cuda_device, dtype, wx, wy, wz):
    a = synth.random_values(np.dtype(dtype), 12 * 40 * 50, seed=wx * 100 + wy * 10 + wz).reshape(12, 40, 50)
    x = torch.from_numpy(a).to(dev())
    mx, mn = mm.maxmin_filter_3d(x, wx, wy, wz)
    torch.cuda.synchronize()
    ex, en = oracle.separable_3d(a, wx, wy, wz)
    assert_same(mx, ex, "3d max")
    assert_same(mn, en, "3d min")


def test_3d_strided_and_single_output(cuda_device):
    a = synth.random_values(np.dtype(np.uint8), 9 * 33 * 64, seed=3).reshape(9, 33, 64)
    x = torch.from_numpy(a).to(dev())
    mx, mn = mm.maxmin_filter_3d(x, 4, 5, 3, cols=57, want_min=False)
    torch.cuda.synchronize()
    assert mn is None
    ex, _ = oracle.separable_3d(np.ascontiguousarray(a[:, :, :57]), 4, 5, 3)
    assert_same(mx, ex, "3d strided max")


@pytest.mark.parametrize("dtype", [np.float32, np.uint8, np.int16], ids=lambda d: np.dtype(d).name)
def test_2d_separable_cropped_batch(cuda_device, dtype):
    """Images cropped from a larger buffer (image stride != rows * row pitch): the
    separable path's per-image row passes; windows outside the packed-byte domain."""
    big = synth.random_values(np.dtype(dtype), 3 * 80 * 96, seed=17).reshape(3, 80, 96)
    x = torch.from_numpy(big).to(dev())[:, 5:69, :]  # 64 rows of each 80-row image: stride 80 * 96
    for wr, wc in [(5, 3), (1, 9), (12, 16), (33, 2)]:
        mx, mn = mm.maxmin_filter_2d(x, wr, wc, cols=90)
        torch.cuda.synchronize()
        ex, en = oracle.separable_2d(np.ascontiguousarray(big[:, 5:69, :90]), wr, wc)
        assert_same(mx, ex, f"max {wr}x{wc}")
        assert_same(mn, en, f"min {wr}x{wc}")


@pytest.mark.parametrize("dtype", [np.float32, np.uint16, np.int8], ids=lambda d: np.dtype(d).name)
def test_2d_plain_entry_generic_kernel(cuda_device, dtype):
    """maxmin_filter_2d (no scratch) through the C ABI: the fused kernels only (packed
    bytes or the generic 2-D kernel), and maxmin_filter_2d_ws without a workspace."""
    import ctypes

    a = synth.random_values(np.dtype(dtype), 2 * 60 * 70, seed=44).reshape(2, 60, 70)
    x = torch.from_numpy(a).to(dev())
    L = mm._lib.lib()
    vp = ctypes.c_void_p
    for wr, wc in [(5, 7), (3, 3), (20, 2)]:
        R, C = 60 - wc + 1, 70 - wr + 1
        ex, en = oracle.separable_2d(a, wr, wc)
        for entry in ("plain", "ws_null"):
            ox = torch.empty(2, R, C, dtype=x.dtype, device=dev())
            on = torch.empty_like(ox)
            args = [mm.dtype_code(x.dtype), vp(x.data_ptr()), 2, 60, 70, 70, 60 * 70, wr, wc, vp(ox.data_ptr()),
                    vp(on.data_ptr()), C, R * C]
            stream = vp(torch.cuda.current_stream().cuda_stream)
            if entry == "plain":
                mm._lib.check(L.maxmin_filter_2d(*args, stream))
            else:
                mm._lib.check(L.maxmin_filter_2d_ws(*args, vp(0), 0, stream))
            torch.cuda.synchronize()
            assert_same(ox, ex, f"{entry} max {wr}x{wc}")
            assert_same(on, en, f"{entry} min {wr}x{wc}")


# ------------------------------------- round 2: SURVEY.md §4 items 2 and 3 ---

@pytest.mark.parametrize("w", [3, 1024, 65536, 262144])
def test_reversal_symmetry(cuda_device, w):
    """F(rev a)[j] = F(a)[n-w-j] at C5's scale (no oracle): the large-window
    kernel's front and the tile seams meet the data in the opposite order."""
    a = synth.c5(1 << 24)
    x = torch.from_numpy(a).to(dev())
    mx, mn = mm.maxmin_filter_1d(x, w)
    rx, rn = mm.maxmin_filter_1d(torch.flip(x, [0]).contiguous(), w)
    assert torch.equal(torch.flip(rx, [0]), mx) and torch.equal(torch.flip(rn, [0]), mn)


@pytest.mark.parametrize("dtype", [np.uint8, np.float32], ids=lambda d: np.dtype(d).name)
@pytest.mark.parametrize("wr,wc", [(15, 15), (5, 11), (17, 3)])
def test_2d_transpose_symmetry(cuda_device, dtype, wr, wc):
    """F_{wr,wc}(A)^T = F_{wc,wr}(A^T) on 2 x 1200 x 1600 images."""
    img = synth.c4(count=2, rows=1200, cols=1600, nrect=5)
    if dtype == np.float32:
        img = img.astype(np.float32)
    x = torch.from_numpy(img).to(dev())
    mx, mn = mm.maxmin_filter_2d(x, wr, wc)
    xt = x.transpose(1, 2).contiguous()
    tx, tn = mm.maxmin_filter_2d(xt, wc, wr)
    assert torch.equal(mx.transpose(1, 2), tx) and torch.equal(mn.transpose(1, 2), tn)


@pytest.mark.parametrize("n", [1, 2, 7, 37, 64, 129])
def test_batched_many_tiny_problems(cuda_device, n):
    """Thousands of tiny random problems in one launch (the batched API), every w,
    against the brute-force definition; tie-heavy values."""
    rows = 4096
    a = synth.random_values(np.int32, rows * n, seed=100 + n, alphabet=8).reshape(rows, n)
    ld = (n + 3) // 4 * 4
    buf = np.zeros((rows, ld), np.int32)
    buf[:, :n] = a
    x = torch.from_numpy(buf).to(dev())
    for w in sorted({1, 2, 3, n // 2 + 1, n}):
        if w > n or w < 1:
            continue
        mx, mn = mm.maxmin_filter_batched(x, w, n=n)
        win = np.lib.stride_tricks.sliding_window_view(a, w, axis=1)
        assert np.array_equal(mx.cpu().numpy(), win.max(axis=2)), (n, w)
        assert np.array_equal(mn.cpu().numpy(), win.min(axis=2)), (n, w)


@pytest.mark.parametrize("dtype", [np.float32, np.uint8, np.int16, np.int32],
                         ids=lambda d: np.dtype(d).name)
@pytest.mark.parametrize("w", [100, 300, 600, 1000, 1024])
def test_medium_direct_gap(cuda_device, dtype, w):
    """k1d_medium's ring-free variant (q' = 0, r' >= 16: each lane group reduces
    its own gap, stages refilled by the last warp done with them): rows of 1-3
    tiles with ragged tails (the shared-memory tail patch), CTA ranges of one or
    two tiles, and repeated launches (the election counters and full barriers
    carry over from tile to tile)."""
    per16 = 16 // np.dtype(dtype).itemsize  # row pitches are whole 16-B vectors (header layout rule)
    for rows, n in ((3, w + 5), (40, 4096 + w - 1), (29, 9000 + w + 13), (5, 3 * 4096 + w + 31)):
        ld = -(-n // per16) * per16
        a = synth.random_values(dtype, rows * ld, seed=w * 7 + rows).reshape(rows, ld)
        x = torch.from_numpy(a).to(dev())
        ex, en = oracle.batched(a, w, n=n)
        for _ in range(3):
            mx, mn = mm.maxmin_filter_batched(x, w, n=n)
            torch.cuda.synchronize()
            assert_same(mx, ex, f"max w={w} rows={rows} n={n}")
            assert_same(mn, en, f"min w={w} rows={rows} n={n}")
