"""Synthetic-input generators (synth/): determinism, preconditions, structure."""
import numpy as np

import synth


def _no_nan_no_negzero(a):
    a = np.asarray(a)
    assert not np.isnan(a).any()
    assert not (np.signbit(a) & (a == 0)).any()


def test_counter_based_subranges():
    full = synth.raw_u64(9, 3, 1000)
    part = synth.raw_u64(9, 3, 100, offset=450)
    assert (full[450:550] == part).all()
    assert (synth.uniform_f32(9, 3, 50, offset=10) == synth.uniform_f32(9, 3, 60)[10:]).all()


def test_c1_c2_c3_preconditions():
    a = synth.c1()
    assert a.shape == (100_000,) and a.dtype == np.float64
    assert (a >= 0).all() and (a < 1).all()
    _no_nan_no_negzero(a)
    w = synth.c2(1 << 16)
    _no_nan_no_negzero(w)
    steps = np.diff(w.astype(np.float64))
    assert abs(steps.mean()) < 0.05 and abs(steps.std() - 1.0) < 0.05  # N(0,1) steps
    assert (synth.c2(1 << 16) == w).all()
    e = synth.c3(rows=16)
    _no_nan_no_negzero(e)
    assert e.shape == (16, 4096) and np.abs(e).max() < 2.0


def test_c4_rectangles():
    img = synth.c4(count=1, rows=512, cols=512, nrect=64)
    assert img.dtype == np.uint8
    # painted rectangles create long constant runs along rows
    runs = (np.diff(img[0].astype(np.int16), axis=1) == 0).mean()
    assert runs > 0.2
    again = synth.c4(count=1, img0=0, rows=512, cols=512, nrect=64)
    assert (again == img).all()


def test_c5_structure():
    n = 1 << 20
    a = synth.c5(n)
    _no_nan_no_negzero(a)
    assert (a >= -1e7).all() and (a < 2 ** 24 + 1).all()
    assert (a == np.round(a)).all()  # integer-valued floats
    d = np.diff(a.astype(np.float64))
    # long strictly monotone runs of step exactly +1 / -1
    assert (d == 1).mean() > 0.15 and (d == -1).mean() > 0.15


def test_edge_values_structure():
    """Edge-case series: every special of the dtype occurs, no NaN / -0, long equal
    runs, deterministic."""
    for dt in (np.uint8, np.int8, np.uint16, np.int16, np.uint32, np.int32, np.uint64, np.int64,
               np.float32, np.float64):
        a = synth.edge_values(dt, 200_000, seed=5)
        assert a.dtype == np.dtype(dt) and a.shape == (200_000,)
        assert np.array_equal(a, synth.edge_values(dt, 200_000, seed=5))
        pool = synth.special_pool(dt)
        assert np.isin(pool, a).all(), np.dtype(dt).name
        if np.dtype(dt).kind == "f":
            _no_nan_no_negzero(a)
            assert np.isinf(a).any() and (np.abs(a[np.isfinite(a)]) < np.finfo(dt).tiny).any()
        runs = np.flatnonzero(np.diff(a.view(f"u{a.dtype.itemsize}")) != 0)
        assert np.diff(runs).max() >= 500  # a long constant run
