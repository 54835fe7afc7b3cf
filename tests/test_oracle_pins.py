"""Pins for the CPU oracle (oracle/), independent of the oracle itself.

Each pin comes from outside the function it checks: worked examples re-derived by
hand (tests/golden, cited), an independent library implementation of the
definition (numpy sliding_window_view + max/min), closed forms, the paper's
invariants (Table 1), exhaustive brute force
on tiny inputs, and metamorphic identities.  No GPU.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
swv = np.lib.stride_tricks.sliding_window_view


def np_filter(a, w):
    """Independent implementation of the definition PAPER.md:39-42 (numpy)."""
    v = swv(np.asarray(a), w)
    return v.max(axis=1), v.min(axis=1)


def np_filter_2d(a, w_row, w_col):
    v = swv(np.asarray(a), (w_col, w_row), axis=(-2, -1))
    return v.max(axis=(-2, -1)), v.min(axis=(-2, -1))


def same(x, y):
    x = np.asarray(x)
    y = np.asarray(y)
    return x.shape == y.shape and x.dtype == y.dtype and x.tobytes() == y.tobytes()


def all_1d(a, w):
    """Every 1-D oracle variant applicable to (a, w): name -> (max, min, stats)."""
    out = {"brute": oracle.brute_1d(a, w), "appendix": oracle.appendix(a, w),
           "vhgw": oracle.vhgw(a, w)}
    if w >= 2:
        out["alg1"] = oracle.alg1(a, w)
    if w == 3:
        out["w3"] = oracle.w3(a)
    return out


# ---------------------------------------------------------------- golden ----

def test_golden_examples_1d():
    g = json.load(open(os.path.join(GOLDEN, "examples_1d.json")))
    for case in g["cases"]:
        a = np.array(case["a"], np.float64)
        for name, (mx, mn, _) in all_1d(a, case["w"]).items():
            assert mx.tolist() == case["max"], (name, case["cite"])
            assert mn.tolist() == case["min"], (name, case["cite"])


def test_golden_naive_count():
    g = json.load(open(os.path.join(GOLDEN, "examples_1d.json")))
    for c in g["counts"]:
        a = synth.uniform_f64(11, 0, c["n"])
        _, _, st = oracle.brute_1d(a, c["w"])
        assert st.comparisons == c["naive_comparisons"], c["cite"]


def test_golden_examples_2d():
    g = json.load(open(os.path.join(GOLDEN, "examples_2d.json")))
    for case in g["cases"]:
        a = np.array(case["a"], np.float64)
        for f in (oracle.brute_2d, oracle.separable_2d):
            mx, mn = f(a, case["w_row"], case["w_col"])
            assert mx.tolist() == case["max"], case["cite"]
            assert mn.tolist() == case["min"], case["cite"]


# ------------------------------------------------- brute force / numpy -----

def test_exhaustive_tiny_alphabet():
    """All arrays of length <= 8 over {0,1,2}, every w (73 812 cases)."""
    count = 0
    for n in range(1, 9):
        for tup in itertools.product((0.0, 1.0, 2.0), repeat=n):
            a = np.array(tup)
            for w in range(1, n + 1):
                ex, en = np_filter(a, w)
                for name, (mx, mn, st) in all_1d(a, w).items():
                    assert same(mx, ex) and same(mn, en), (name, tup, w)
                    if name in ("alg1", "appendix"):
                        assert st.comparisons <= 3 * n, (name, tup, w)
                        assert st.peak_wedge <= w + 1, (name, tup, w)
                count += 1
    assert count == 73812


@pytest.mark.parametrize("alphabet", [None, 8])
def test_random_cases_vs_numpy(alphabet):
    """SPEC.md:397 recipe: 1000 cases, n in [1,256], w in [1,n], continuous and {0..7}."""
    for k in range(1000):
        n = 1 + synth.rng(21, 0, k) % 256
        w = 1 + synth.rng(21, 1, k) % n
        a = synth.random_values(np.float64, n, seed=22 + k, alphabet=alphabet)
        ex, en = np_filter(a, w)
        for name, (mx, mn, st) in all_1d(a, w).items():
            assert same(mx, ex) and same(mn, en), (name, n, w, k)


@pytest.mark.parametrize("dtype", oracle.DTYPES)
def test_every_dtype_vs_numpy(dtype):
    """Full-range values (incl. > 2^53 for 64-bit ints, negative floats)."""
    for k, (n, w) in enumerate([(1, 1), (7, 3), (300, 17), (1000, 1000), (4097, 129)]):
        a = synth.random_values(dtype, n, seed=31 + k)
        ex, en = np_filter(a, w)
        mx, mn, _ = oracle.appendix(a, w)
        assert same(mx, ex) and same(mn, en), (dtype, n, w)
        mx, mn, _ = oracle.brute_1d(a, w)
        assert same(mx, ex) and same(mn, en), (dtype, n, w)
    info = np.iinfo(dtype) if np.dtype(dtype).kind in "iu" else np.finfo(dtype)
    a = np.array([info.max, info.min, 0, info.max, info.min], dtype)
    ex, en = np_filter(a, 2)
    mx, mn, _ = oracle.appendix(a, 2)
    assert same(mx, ex) and same(mn, en)


def test_windows_at_and_batched_vs_numpy():
    a = synth.random_values(np.float32, 5000, seed=41)
    starts = np.array([0, 1, 17, 4000, 5000 - 300], np.int64)
    mx, mn = oracle.windows_at(a, 300, starts)
    ex, en = np_filter(a, 300)
    assert same(mx, ex[starts]) and same(mn, en[starts])
    b = synth.random_values(np.float32, 7 * 200, seed=42).reshape(7, 200)
    mx, mn = oracle.batched(b, 33)
    for r in range(7):
        ex, en = np_filter(b[r], 33)
        assert same(mx[r], ex) and same(mn[r], en)


# ------------------------------------------------------------ closed forms --

def test_closed_forms():
    n = 1000
    up = synth.ramp_up(n)
    down = synth.ramp_down(n)
    for w in (1, 2, 3, 10, 999, 1000):
        for name, (mx, mn, _) in all_1d(up, w).items():  # non-decreasing
            assert same(mx, up[w - 1:]) and same(mn, up[: n - w + 1]), name
        for name, (mx, mn, _) in all_1d(down, w).items():  # non-increasing
            assert same(mx, down[: n - w + 1]) and same(mn, down[w - 1:]), name
        c = synth.constant(n, 7.0)
        for name, (mx, mn, _) in all_1d(c, w).items():
            assert (mx == 7.0).all() and (mn == 7.0).all(), name
    a = synth.uniform_f64(5, 0, n)
    for name, (mx, mn, _) in all_1d(a, 1).items():  # w = 1: identity
        assert same(mx, a) and same(mn, a), name
    for name, (mx, mn, _) in all_1d(a, n).items():  # w = n: global max/min
        assert mx.tolist() == [a.max()] and mn.tolist() == [a.min()], name
    alt = synth.alternating(n)
    for w in (2, 3, 50):
        for name, (mx, mn, _) in all_1d(alt, w).items():
            assert (mx == 1.0).all() and (mn == 0.0).all(), name


# -------------------------------------------------------------- invariants --

FAMILIES = {
    "uniform": lambda n: synth.uniform_f64(3, 0, n),
    "sine": lambda n: synth.sine(n, 10000),
    "ramp_up": synth.ramp_up,
    "ramp_down": synth.ramp_down,
    "constant": lambda n: synth.constant(n, 7.0),
    "alternating": synth.alternating,
    "piecewise": lambda n: synth.piecewise(n, 40, seed=4),
    "tie_alphabet": lambda n: synth.random_values(np.float64, n, seed=6, alphabet=8),
}


@pytest.mark.parametrize("family", sorted(FAMILIES))
def test_comparison_bounds(family):
    """Prop. PAPER.md:406-410 (<= 3n), Prop. PAPER.md:477-479 (<= 2n if monotone),
    Prop. PAPER.md:494-497 (size(U)+size(L) <= w+1); SPEC.md:398-403 grid."""
    n = 100_000
    a = FAMILIES[family](n)
    monotone = family in ("ramp_up", "ramp_down", "constant")
    for w in (3, 10, 100, 1000, 10_000):
        ex, en = np_filter(a, w)
        for f in (oracle.alg1, oracle.appendix):
            mx, mn, st = f(a, w)
            assert same(mx, ex) and same(mn, en)
            assert st.comparisons <= 3 * n
            assert st.peak_wedge <= w + 1
            if monotone:
                assert st.comparisons <= 2 * n
                # hand derivation: on a monotone input each loop step does the
                # line-379 comparison and the while loop never runs
                assert st.comparisons == n - 1


def test_iid_cost_approaches_three():
    """Survey measurement: i.i.d. input at w=1000 costs
    ~2.996 comparisons per element -- close to, never above, the bound 3."""
    n = 100_000
    a = synth.uniform_f64(3, 0, n)
    _, _, st = oracle.alg1(a, 1000)
    assert 2.95 < st.comparisons / n <= 3.0


def test_naive_count_formula():
    """Table 1 naive row (2w-2 per element), exact."""
    n = 1000
    a = synth.uniform_f64(7, 0, n)
    for w in (1, 2, 10, 100, 1000):
        _, _, st = oracle.brute_1d(a, w)
        assert st.comparisons == (n - w + 1) * 2 * (w - 1)


def test_vhgw_bound():
    """Table 1: van Herk-Gil-Werman <= 6-8/w comparisons per element on
    block-aligned inputs."""
    for w in (4, 16, 64):
        n = 100 * w
        for fam in ("uniform", "sine", "alternating", "ramp_up"):
            a = FAMILIES[fam](n)
            mx, mn, st = oracle.vhgw(a, w)
            ex, en = np_filter(a, w)
            assert same(mx, ex) and same(mn, en)
            assert st.comparisons <= (6 - 8 / w) * n


def test_w3_two_comparisons():
    """Proposition: w = 3 in <= 2 comparisons per element."""
    n = 100_000
    for fam in sorted(FAMILIES):
        a = FAMILIES[fam](n)
        mx, mn, st = oracle.w3(a)
        ex, en = np_filter(a, 3)
        assert same(mx, ex) and same(mn, en), fam
        assert st.comparisons <= 2 * n


# ------------------------------------------------------------------ 2-D -----

def test_2d_separable_equals_rectangles():
    """50 seeded 64x64 grids, (w_row, w_col) in {1..8}^2."""
    for g in range(50):
        a = synth.random_values(np.float32, 64 * 64, seed=100 + g,
                                alphabet=16 if g % 2 else None).reshape(64, 64)
        pairs = [(wr, wc) for wr in range(1, 9) for wc in range(1, 9)]
        if g >= 4:  # all 64 pairs on 4 grids, 8 seeded pairs on the rest
            pairs = [pairs[synth.rng(101, g, k) % 64] for k in range(8)]
        for wr, wc in pairs:
            ex, en = np_filter_2d(a, wr, wc)
            bx, bn = oracle.brute_2d(a, wr, wc)
            sx, sn = oracle.separable_2d(a, wr, wc)
            assert same(bx, ex) and same(bn, en), (g, wr, wc)
            assert same(sx, ex) and same(sn, en), (g, wr, wc)


def test_2d_transpose_symmetry_and_batch():
    a = synth.c4(count=2, rows=70, cols=90, nrect=5)
    mx, mn = oracle.separable_2d(a, 5, 9)
    tx, tn = oracle.separable_2d(np.ascontiguousarray(a.transpose(0, 2, 1)), 9, 5)
    assert same(mx, np.ascontiguousarray(tx.transpose(0, 2, 1)))
    assert same(mn, np.ascontiguousarray(tn.transpose(0, 2, 1)))
    for b in range(2):
        ex, en = np_filter_2d(a[b], 5, 9)
        assert same(mx[b], ex) and same(mn[b], en)


# --------------------------------------------------------------- errors -----

def test_errors():
    a = np.arange(5, dtype=np.float64)
    for f in (oracle.brute_1d, oracle.appendix, oracle.vhgw, oracle.alg1):
        with pytest.raises(oracle.OracleError) as e:
            f(a, 0)
        assert e.value.code == -1
        with pytest.raises(oracle.OracleError) as e:
            f(a, 6)
        assert e.value.code == -2
    b = a.copy()
    b[2] = np.nan
    for f in (oracle.brute_1d, oracle.appendix, oracle.alg1, oracle.vhgw):
        with pytest.raises(oracle.OracleError) as e:
            f(b, 2)
        assert e.value.code == -3
    with pytest.raises(oracle.OracleError):
        oracle.alg1(a, 1)  # reading R4: Algorithm 1 needs w >= 2
    with pytest.raises(oracle.OracleError):
        oracle.brute_2d(np.zeros((3, 3)), 4, 1)


# ------------------------------------------------------------ N1: arg filter
# Pins for oracle_arg_brute / oracle_arg_wedge: printed
# examples, numpy's argmax/argmin (an independent implementation that returns
# the FIRST occurrence -- the earliest-position rule R17), and the wedge equal
# to the definition on every tiny case.

def test_golden_arg_examples():
    cases = json.load(open(os.path.join(GOLDEN, "examples_1d.json")))["arg_cases"]
    for c in cases:
        a = np.array(c["a"], np.int32)
        for fn in (oracle.arg_brute, oracle.arg_wedge):
            mx, mn, ax, an = fn(a, c["w"])
            assert ax.tolist() == c["argmax"], (c["cite"], fn.__name__)
            assert an.tolist() == c["argmin"], (c["cite"], fn.__name__)
            assert mx.tolist() == a[ax].tolist() and mn.tolist() == a[an].tolist()


@pytest.mark.parametrize("dtype", [np.uint8, np.int8, np.int16, np.uint32, np.int32, np.float32, np.float64])
def test_arg_vs_numpy(dtype):
    rng = np.random.default_rng(17)
    for t in range(60):
        n = int(rng.integers(1, 300))
        w = int(rng.integers(1, n + 1))
        a = synth.random_values(dtype, n, seed=500 + t, alphabet=(3 if t % 2 else None))
        win = np.lib.stride_tricks.sliding_window_view(a, w)
        base = np.arange(n - w + 1)
        for fn in (oracle.arg_brute, oracle.arg_wedge):
            mx, mn, ax, an = fn(a, w)
            assert np.array_equal(ax, base + win.argmax(axis=1)), (t, fn.__name__)
            assert np.array_equal(an, base + win.argmin(axis=1)), (t, fn.__name__)
            assert np.array_equal(mx, win.max(axis=1)) and np.array_equal(mn, win.min(axis=1))


def test_arg_wedge_equals_brute_exhaustive():
    for n in range(1, 8):
        for code in range(3 ** n):
            a = np.array([(code // 3 ** k) % 3 for k in range(n)], np.int32)
            for w in range(1, n + 1):
                b = oracle.arg_brute(a, w)
                g = oracle.arg_wedge(a, w)
                for x, y in zip(b, g):
                    assert np.array_equal(x, y), (a.tolist(), w)


# ------------------------------------------------------------ N3: LB_Keogh
# Pins for oracle_keogh_f32: the envelope equals scipy's
# maximum/minimum_filter1d with edge replication (an independent library
# implementation of the clipped window, reading R18); the bound equals the
# formula recomputed from that envelope; LB_Keogh lower-bounds the banded DTW
# distance (its defining property, computed here by brute-force dynamic
# programming); it is 0 against itself and non-increasing in r.

def _dtw_band(a, b, r):
    n = len(a)
    D = np.full((n + 1, n + 1), np.inf)
    D[0, 0] = 0.0
    for i in range(1, n + 1):
        for j in range(max(1, i - r), min(n, i + r) + 1):
            d = (float(a[i - 1]) - float(b[j - 1])) ** 2
            D[i, j] = d + min(D[i - 1, j], D[i, j - 1], D[i - 1, j - 1])
    return np.sqrt(D[n, n])


def test_keogh_envelope_vs_scipy_and_formula():
    from scipy.ndimage import maximum_filter1d, minimum_filter1d
    rng = np.random.default_rng(23)
    for t in range(40):
        n = int(rng.integers(1, 200))
        r = int(rng.integers(0, n + 3))
        c = rng.standard_normal((3, n)).astype(np.float32)
        q = rng.standard_normal(n).astype(np.float32)
        lb, U, L = oracle.keogh(c, q, r, envelope=True)
        lbb = oracle.keogh(c, q, r, brute=True)
        assert np.array_equal(lb, lbb)
        for b in range(3):
            eu = maximum_filter1d(c[b], size=2 * r + 1, mode="nearest")
            el = minimum_filter1d(c[b], size=2 * r + 1, mode="nearest")
            assert np.array_equal(U[b], eu) and np.array_equal(L[b], el), (t, n, r)
            qd, ud, ld = q.astype(np.float64), eu.astype(np.float64), el.astype(np.float64)
            s = np.where(qd > ud, (qd - ud) ** 2, np.where(qd < ld, (ld - qd) ** 2, 0.0)).sum()
            assert abs(lb[b] - np.sqrt(s)) <= 1e-12 * max(1.0, np.sqrt(s))


def test_keogh_lower_bounds_dtw():
    rng = np.random.default_rng(29)
    for t in range(60):
        n = int(rng.integers(2, 40))
        r = int(rng.integers(0, n))
        a = np.cumsum(rng.standard_normal(n)).astype(np.float32)
        b = np.cumsum(rng.standard_normal(n)).astype(np.float32)
        lb = oracle.keogh(b[None], a, r)[0]  # envelope around the candidate b, query a
        assert lb <= _dtw_band(a, b, r) * (1 + 1e-9) + 1e-12, (t, n, r)


def test_keogh_identity_and_monotone_in_r():
    c = synth.c3(rows=4, length=300)
    for b in range(4):
        assert oracle.keogh(c[b][None], c[b], 5)[0] == 0.0
    q = synth.c3(rows=1, length=300, row0=99)[0]
    prev = np.inf
    for r in (0, 1, 2, 4, 8, 16, 64, 299):
        lb = oracle.keogh(c, q, r)
        assert np.all(lb <= prev)
        prev = lb


# ---------------------------------------------------------------- N2 streaming
def _stream_all(a, w, sizes, dtype=None):
    s = oracle.Stream(np.asarray(a).dtype if dtype is None else dtype, w)
    outs, off = [], 0
    for c in sizes:
        outs.append(s.push(np.asarray(a)[off:off + c]))
        off += c
    return s, outs


def test_stream_spec_examples():
    """w=3 pushes 1,3,2 -> (3, 1) on the third push only; 2,2,2 -> (2, 2);
    w=1 emits on the first push."""
    s = oracle.Stream(np.int64, 3)
    assert [len(s.push([v])[0]) for v in (1, 3)] == [0, 0]
    mx, mn = s.push([2])
    assert mx.tolist() == [3] and mn.tolist() == [1]
    s = oracle.Stream(np.int64, 3)
    mx, mn = s.push([2, 2, 2])
    assert mx.tolist() == [2] and mn.tolist() == [2]
    s = oracle.Stream(np.int64, 1)
    mx, mn = s.push([5])
    assert mx.tolist() == [5] and mn.tolist() == [5]


def test_stream_exhaustive_tiny_zero_latency():
    """Every {0,1,2}^n, n <= 6, every w, pushes of every composition of n into <= 3 parts:
    concatenated emissions = the definition (numpy); each push emits exactly the windows
    its samples complete (zero stream latency)."""
    for n in range(1, 7):
        comps = [(n,)] + [(k, n - k) for k in range(0, n + 1)] + [(1, k, n - 1 - k) for k in range(0, n)]
        for a in itertools.product(range(3), repeat=n):
            a = np.array(a, np.int32)
            for w in range(1, n + 2):
                for sizes in comps:
                    _, outs = _stream_all(a, w, sizes)
                    seen = 0
                    for (mx, mn), c in zip(outs, sizes):
                        want = max(0, seen + c - w + 1) - max(0, seen - w + 1)
                        assert len(mx) == want, (a, w, sizes)
                        seen += c
                    got_x = np.concatenate([o[0] for o in outs])
                    got_n = np.concatenate([o[1] for o in outs])
                    if w <= n:
                        ex, en = np_filter(a, w)
                        assert same(got_x, ex) and same(got_n, en), (a, w, sizes)
                    else:
                        assert len(got_x) == 0


@pytest.mark.parametrize("dtype", oracle.DTYPES)
def test_stream_random_chunks_vs_numpy(dtype):
    rng = np.random.default_rng(7)
    a = synth.random_values(np.dtype(dtype), 3000, seed=11)
    for w in (1, 2, 5, 64, 700):
        sizes = rng.integers(0, 300, size=40)
        sizes = sizes[np.cumsum(sizes) <= a.shape[0]]
        n = int(sizes.sum())
        _, outs = _stream_all(a, w, sizes.tolist())
        ex, en = np_filter(a[:n], w)
        assert same(np.concatenate([o[0] for o in outs]), ex)
        assert same(np.concatenate([o[1] for o in outs]), en)


@pytest.mark.parametrize("family", ["increasing", "decreasing", "alternating", "uniform"])
def test_stream_comparison_and_wedge_bounds(family):
    """Propositions PAPER.md:406-505 hold across push boundaries: <= 3n comparisons (<= 2n
    on monotone input) and size(U)+size(L) <= w+1."""
    n = 20000
    rng = np.random.default_rng(3)
    a = {"increasing": np.arange(n, dtype=np.float64), "decreasing": -np.arange(n, dtype=np.float64),
         "alternating": (np.arange(n) % 2).astype(np.float64), "uniform": rng.random(n)}[family]
    for w in (2, 3, 17, 1000):
        sizes = [97] * (n // 97) + [n % 97]
        s, _ = _stream_all(a, w, sizes)
        st = s.stats()
        assert st.comparisons <= 3 * n
        if family in ("increasing", "decreasing"):
            assert st.comparisons <= 2 * n
        assert st.peak_wedge <= w + 1


# ---------------------------------------------------------------- N4 morphology
def test_morph_exhaustive_brute_equals_composition():
    """Every {0,1,2}^n, n <= 7, every w <= n: the definition (R20) = the composition."""
    for n in range(1, 8):
        for a in itertools.product(range(3), repeat=n):
            a = np.array(a, np.int16)
            for w in range(1, n + 1):
                bo, bc = oracle.morph(a, w, brute=True)
                co, cc = oracle.morph(a, w)
                assert same(bo, co) and same(bc, cc), (a, w)


def test_morph_hand_examples():
    """Opening removes peaks narrower than w and keeps plateaus of width >= w; closing
    fills narrow valleys (worked by hand)."""
    a = np.array([0, 0, 5, 0, 0, 7, 7, 7, 0, 0], np.int32)
    op, cl = oracle.morph(a, 3, brute=True)
    assert op.tolist() == [0, 0, 0, 0, 0, 7, 7, 7, 0, 0]
    assert cl.tolist() == [5, 5, 5, 5, 5, 7, 7, 7, 7, 7]  # windows stay inside: the ends are filled too
    b = np.array([4, 4, 1, 4, 4, 4], np.int32)
    op, cl = oracle.morph(b, 2, brute=True)
    assert cl.tolist() == [4, 4, 4, 4, 4, 4]  # the width-1 valley is filled
    assert op.tolist() == [4, 4, 1, 4, 4, 4]


@pytest.mark.parametrize("dtype", oracle.DTYPES)
def test_morph_properties_and_scipy(dtype):
    """Anti-extensive opening, extensive closing, idempotence, and scipy.ndimage
    grey_opening / grey_closing away from the borders (the operators are translation
    invariant, so the origin convention cancels in the interior)."""
    from scipy import ndimage

    a = synth.random_values(np.dtype(dtype), 4000, seed=21)
    for w in (1, 2, 5, 16, 33):
        op, cl = oracle.morph(a, w)
        assert np.all(op <= a) and np.all(cl >= a)
        op2, _ = oracle.morph(op, w)
        _, cl2 = oracle.morph(cl, w)
        assert same(op2, op) and same(cl2, cl)
        if np.dtype(dtype).itemsize == 8 and np.dtype(dtype).kind in "iu":
            continue  # scipy.ndimage computes 64-bit integers through float64
        so = ndimage.grey_opening(a, size=w)
        sc = ndimage.grey_closing(a, size=w)
        lo, hi = 2 * w, a.shape[0] - 2 * w
        assert same(op[lo:hi], so[lo:hi]) and same(cl[lo:hi], sc[lo:hi])


def test_morph_duality_f64():
    a = synth.random_values(np.dtype(np.float64), 3000, seed=4)
    for w in (3, 40):
        op, cl = oracle.morph(a, w)
        nop, ncl = oracle.morph(-a, w)
        assert same(cl, -nop) and same(op, -ncl)


def test_morph_2d_brute_and_scipy():
    from scipy import ndimage

    rng = np.random.default_rng(9)
    for (rows, cols, wr, wc) in [(5, 6, 2, 3), (7, 7, 3, 3), (4, 9, 4, 1), (6, 5, 1, 2), (8, 8, 8, 8)]:
        a = rng.integers(0, 4, size=(2, rows, cols)).astype(np.uint8)
        bo, bc = oracle.morph_2d(a, wr, wc, brute=True)
        co, cc = oracle.morph_2d(a, wr, wc)
        assert same(bo, co) and same(bc, cc), (rows, cols, wr, wc)
    a = synth.random_values(np.dtype(np.uint8), 120 * 130, seed=3).reshape(120, 130)
    op, cl = oracle.morph_2d(a, 5, 7)
    so = ndimage.grey_opening(a, size=(7, 5))
    sc = ndimage.grey_closing(a, size=(7, 5))
    assert same(op[14:-14, 10:-10], so[14:-14, 10:-10]) and same(cl[14:-14, 10:-10], sc[14:-14, 10:-10])
    r1o, r1c = oracle.morph(a[3], 5)  # one row, w_col = 1: the 1-D operators
    o1, c1 = oracle.morph_2d(a[3:4], 5, 1)
    assert same(o1[0], r1o) and same(c1[0], r1c)


# ---------------------------------------------------------- N4: 3-D filters
def test_3d_brute_equals_separable():
    rng = np.random.default_rng(5)
    for (d, r, c, wx, wy, wz) in [(4, 5, 6, 2, 3, 2), (3, 3, 3, 3, 3, 3), (5, 4, 7, 1, 1, 5), (6, 2, 9, 4, 2, 1),
                                  (7, 6, 5, 5, 6, 3)]:
        for dt in (np.uint8, np.int32, np.float64):
            a = rng.integers(0, 4, size=(d, r, c)).astype(dt)
            bx, bn = oracle.brute_3d(a, wx, wy, wz)
            sx, sn = oracle.separable_3d(a, wx, wy, wz)
            assert same(bx, sx) and same(bn, sn), (d, r, c, wx, wy, wz, dt)


def test_3d_vs_numpy_and_2d():
    a = synth.random_values(np.dtype(np.float32), 9 * 20 * 23, seed=8).reshape(9, 20, 23)
    v = swv(a, (3, 4, 5), axis=(0, 1, 2))  # windows of w_z=3, w_y=4, w_x=5
    mx, mn = oracle.separable_3d(a, 5, 4, 3)
    assert same(mx, v.max(axis=(-3, -2, -1))) and same(mn, v.min(axis=(-3, -2, -1)))
    m2x, m2n = oracle.separable_2d(a, 5, 4)  # w_z = 1 is the 2-D filter of every slice
    m3x, m3n = oracle.separable_3d(a, 5, 4, 1)
    assert same(m2x, m3x) and same(m2n, m3n)


def test_oracle_on_edge_values_vs_numpy():
    """Extremes, +-inf, subnormals and long equal runs: the oracle's streaming
    variants equal numpy's sliding-window max/min bit for bit."""
    import synth

    for dt in (np.uint8, np.int8, np.int16, np.uint32, np.int64, np.float32, np.float64):
        a = synth.edge_values(dt, 30_000, seed=9)
        for w in (1, 2, 3, 17, 300, 4000):
            win = swv(a, w)
            ex, en = win.max(axis=1), win.min(axis=1)
            for f in (oracle.appendix, oracle.alg1) if w >= 2 else (oracle.appendix,):
                mx, mn, _ = f(a, w)
                assert np.array_equal(mx.view(f"u{a.dtype.itemsize}"), ex.view(f"u{a.dtype.itemsize}")), (dt, w)
                assert np.array_equal(mn.view(f"u{a.dtype.itemsize}"), en.view(f"u{a.dtype.itemsize}")), (dt, w)


def test_appendix_baseline_build_equals_oracle():
    """The CPU-baseline build (-O3 -march=native, threads over window ranges) computes
    what the pinned oracle computes."""
    import synth

    a = synth.c5(1_000_003)
    for w in (1, 7, 4096, 262144):
        ex, en, _ = oracle.appendix(a, w)
        for th in (1, 3, 8):
            mx, mn = oracle.appendix_baseline(a, w, th)
            assert np.array_equal(mx, ex) and np.array_equal(mn, en), (w, th)
