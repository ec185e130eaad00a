"""The C restatement (oracle/oracle.c) is pinned against the reference: golden vectors the
reference CPU executor produced (tests/golden/kernels.npz, oracle/make_golden.py) and, where
the reference build is present, live reference runs at other sizes."""
import ctypes as C
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
F = C.POINTER(C.c_float)
I32 = C.POINTER(C.c_int32)
I64 = C.POINTER(C.c_int64)


@pytest.fixture(scope="module")
def g():
    return dict(np.load(os.path.join(GOLDEN, "kernels.npz")))


def heat(okern, a, iters, alpha=0.1):
    rows, cols = a.shape
    cur, nxt = a.copy(), np.empty_like(a)
    for _ in range(iters):
        okern.oracle_heat2d(C.c_int64(rows), C.c_int64(cols), C.c_double(alpha), cur.ctypes.data_as(F), nxt.ctypes.data_as(F))
        cur, nxt = nxt, cur
    return cur


def test_ramp_and_heat2d_match_golden(okern, g):
    rows, cols = g["heat_in"].shape
    a = np.empty((rows, cols), np.float32)
    okern.oracle_ramp2d_f32(C.c_int64(rows), C.c_int64(cols), C.c_int64(1000), C.c_double(0.0), C.c_double(1.0), a.ctypes.data_as(F))
    assert np.array_equal(a, g["heat_in"])
    assert np.array_equal(heat(okern, a, 3).view(np.uint32), g["heat_out"].view(np.uint32))


def test_heat2d_row_band_equals_full_step(okern, g):
    a = g["heat_in"]
    rows, cols = a.shape
    full = heat(okern, a, 1)
    band = np.empty((10, cols), np.float32)
    # rows [12, 22) from an input band holding rows [11, 23)
    src = np.ascontiguousarray(a[11:23])
    okern.oracle_heat2d_rows(C.c_int64(rows), C.c_int64(cols), C.c_double(0.1), src.ctypes.data_as(F), C.c_int64(11), C.c_int64(12),
                             band.ctypes.data_as(F), C.c_int64(12), C.c_int64(22))
    assert np.array_equal(band, full[12:22])


def test_histogram_matches_golden(okern, g):
    n, bins = g["hist_x"].size, g["hist_out"].size
    x = np.empty(n, np.int32)
    okern.oracle_hpattern1d(C.c_int64(0), C.c_int64(n), C.c_int64(bins), C.c_int64(12345), x.ctypes.data_as(I32))
    assert np.array_equal(x, g["hist_x"])
    h = np.empty(bins, np.int64)
    okern.oracle_histogram(x.ctypes.data_as(I32), C.c_int64(n), C.c_int64(bins), h.ctypes.data_as(I64))
    assert np.array_equal(h, g["hist_out"])
    h2 = np.empty(bins, np.int64)
    okern.oracle_histogram_hashed(C.c_int64(0), C.c_int64(n), C.c_int64(bins), C.c_int64(12345), h2.ctypes.data_as(I64))
    assert np.array_equal(h2, h)


def test_kmeans_i32_matches_golden(okern, g):
    pts = g["km_points"]
    n, d = pts.shape
    k = g["km_centroids"].shape[0]
    cen = np.empty((k, d), np.int32)
    okern.oracle_ipattern2d_i32(C.c_int64(k), C.c_int64(d), C.c_int64(997), cen.ctypes.data_as(I32))
    p2 = np.empty_like(pts)
    okern.oracle_ipattern2d_i32(C.c_int64(n), C.c_int64(d), C.c_int64(1000), p2.ctypes.data_as(I32))
    assert np.array_equal(p2, pts)
    asg = np.empty(n, np.int32)
    sums = np.empty((k, d), np.int64)
    cnts = np.empty(k, np.int64)
    for _ in range(3):
        okern.oracle_kmeans_assign_i32(C.c_int64(n), C.c_int64(k), C.c_int64(d), pts.ctypes.data_as(I32), cen.ctypes.data_as(I32), asg.ctypes.data_as(I32))
        okern.oracle_kmeans_update_i32(C.c_int64(n), C.c_int64(k), C.c_int64(d), pts.ctypes.data_as(I32), asg.ctypes.data_as(I32), sums.ctypes.data_as(I64),
                                       cnts.ctypes.data_as(I64))
        okern.oracle_kmeans_finalize_i32(C.c_int64(k), C.c_int64(d), sums.ctypes.data_as(I64), cnts.ctypes.data_as(I64), cen.ctypes.data_as(I32))
    assert np.array_equal(asg, g["km_assign"])
    assert np.array_equal(sums, g["km_sums"])
    assert np.array_equal(cnts, g["km_counts"])
    assert np.array_equal(cen, g["km_centroids"])


def test_heat2d_matches_live_reference_executor(okern, ref):
    """A different size and a 1x3 system: the reference executor vs the C restatement."""
    import oracle
    from paper_2202_05549_b200 import Arr
    rows, cols, iters = 57, 33, 4
    ctx = oracle.reference_context(workers=1, devices=3, execute=True)
    devs = ctx.devices
    dist = lambda: ctx.dist.stencil([rows, cols], [19, 11], [1, 1], devs)  # noqa: E731
    a = ctx.create_array([rows, cols], "f32", dist(), 0)
    b = ctx.create_array([rows, cols], "f32", dist(), 0)
    w = ctx.dist.block_work([rows, cols], [19, 11], [19, 11], devs)
    ctx.launch("ramp2d_f32", [rows, cols], [19, 11], w, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
    for _ in range(iters):
        ctx.launch("heat2d", [rows, cols], [19, 11], w, [rows, cols, 0.1, Arr(b), Arr(a)], "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]")
        a, b = b, a
    got = ctx.read(a)
    ctx.close()
    init = np.empty((rows, cols), np.float32)
    okern.oracle_ramp2d_f32(C.c_int64(rows), C.c_int64(cols), C.c_int64(1000), C.c_double(0.0), C.c_double(1.0), init.ctypes.data_as(F))
    assert np.array_equal(heat(okern, init, iters).view(np.uint32), got.view(np.uint32))
