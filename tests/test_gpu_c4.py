"""C4 kernels at sizes beyond the golden vectors: histogram paths (shared u32, packed u16 pairs,
global), k-means fast/exact paths, all bit-exact against the C oracle."""
import ctypes as C

import numpy as np
import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr

pytestmark = pytest.mark.gpu
I32 = C.POINTER(C.c_int32)
I64 = C.POINTER(C.c_int64)


@pytest.mark.parametrize("bins", [7, 256, 16384, 16385, 65536, 100000, 110001, 220000, 300000])
def test_histogram_paths(okern, bins):
    n = 3_000_017
    with mb.context(workers=1, devices=2, num_gpus=1) as ctx:
        devs = ctx.devices
        x = ctx.create_array([n], "i32", ctx.dist.row([n], 1_500_160, devs), 0)
        h = ctx.create_array([bins], "i64", ctx.dist.replicated([bins], devs), 0)
        w = ctx.dist.block_work([n], [128], [1_500_160], devs)
        ctx.launch("hpattern1d", [n], [128], w, [n, bins, 99, Arr(x)], "global i => write out[i]")
        ctx.launch("histogram", [n], [128], w, [n, bins, Arr(x), Arr(h)], "global i => read x[i], reduce(+) hist[:]")
        got = ctx.read(h)
    want = np.empty(bins, np.int64)
    okern.oracle_histogram_hashed(C.c_int64(0), C.c_int64(n), C.c_int64(bins), C.c_int64(99), want.ctypes.data_as(I64))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("bins", [256, 16385, 65536, 110001, 220000])
def test_histogram_out_of_range_values(okern, bins):
    """values below 0 and at or above `bins` are skipped (oracle_histogram), mixed into the
    in-range ones at every position of the 16-byte loads (the batched kernels test four values
    at a time and fall back per element), plus a hot bin that wraps the shared counters; n not a
    multiple of 4 (the scalar tail)"""
    n = 5_000_003
    rng = np.random.default_rng(bins)
    x = rng.integers(0, bins, size=n, dtype=np.int64)
    x[rng.random(n) < 0.02] = bins + rng.integers(0, 1000, size=1)[0]
    x[rng.random(n) < 0.02] = -1 - rng.integers(0, 1 << 30, size=1)[0]
    x[::7] = 3  # hot bin
    x[-5:] = [bins, -1, 0, bins - 1, (1 << 31) - 1]
    x = x.astype(np.int32)
    with mb.context(workers=1, devices=1, num_gpus=1) as ctx:
        d = ctx.devices
        xa = ctx.create_array([n], "i32", ctx.dist.single([n], d[0]), 0)
        h = ctx.create_array([bins], "i64", ctx.dist.single([bins], d[0]), 0)
        ctx.write(xa, x)
        ctx.launch("histogram", [n], [128], ctx.dist.block_work([n], [128], [-(-n // 128) * 128], d), [n, bins, Arr(xa), Arr(h)],
                   "global i => read x[i], reduce(+) hist[:]")
        got = ctx.read(h)
    want = np.empty(bins, np.int64)
    okern.oracle_histogram(x.ctypes.data_as(I32), C.c_int64(n), C.c_int64(bins), want.ctypes.data_as(I64))
    assert np.array_equal(got, want)


def test_histogram_u16_overflow():
    """every element in one bin: the packed-u16 counters wrap many times"""
    n, bins = 1 << 20, 65536
    with mb.context(workers=1, devices=1, num_gpus=1) as ctx:
        d = ctx.devices
        x = ctx.create_array([n], "i32", ctx.dist.single([n], d[0]), 1)  # all ones -> bin 1
        h = ctx.create_array([bins], "i64", ctx.dist.single([bins], d[0]), 0)
        ctx.launch("histogram", [n], [128], ctx.dist.block_work([n], [128], [n], d), [n, bins, Arr(x), Arr(h)], "global i => read x[i], reduce(+) hist[:]")
        got = ctx.read(h)
    assert got[1] == n and got.sum() == n


@pytest.mark.parametrize("pattern", ["pair", "lo_heavy", "hi_heavy", "odd_bins"])
def test_histogram_u16_wraps_in_shared_words(pattern):
    """two hot bins sharing one packed word (a low half whose carries land in a hot high half),
    both wrapping many times in every CTA: exact counts"""
    n = 1 << 26
    i = np.arange(n, dtype=np.int64)
    bins = 65536 if pattern != "odd_bins" else 65535
    if pattern == "pair":
        x = (2 + (i & 1)).astype(np.int32)                    # bins 2 and 3 alternate
    elif pattern == "lo_heavy":
        x = np.where(i % 5 == 0, 7, 6).astype(np.int32)       # bin 6 (low half) 4x as hot as bin 7
    elif pattern == "hi_heavy":
        x = np.where(i % 5 == 0, 6, 7).astype(np.int32)
    else:
        x = np.where(i % 3 == 0, 65533, 65534).astype(np.int32)  # last word's high half is no bin
    want = np.bincount(x, minlength=bins).astype(np.int64)
    with mb.context(workers=1, devices=1, num_gpus=1) as ctx:
        d = ctx.devices
        xa = ctx.create_array([n], "i32", ctx.dist.single([n], d[0]), 0)
        h = ctx.create_array([bins], "i64", ctx.dist.single([bins], d[0]), 0)
        ctx.write(xa, x)
        ctx.launch("histogram", [n], [256], ctx.dist.block_work([n], [256], [n], d), [n, bins, Arr(xa), Arr(h)], "global i => read x[i], reduce(+) hist[:]")
        got = ctx.read(h)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("mod", [1000, 20000])
def test_kmeans_fast_and_exact_paths(okern, mod):
    """mod 1000: all coordinates < 8192 (u32 fast path); mod 20000: int64 path."""
    n, k, d = 50_000, 64, 16
    with mb.context(workers=1, devices=2, num_gpus=1) as ctx:
        devs = ctx.devices
        pts = ctx.create_array([n, d], "i32", ctx.dist.row([n, d], 25_000, devs), 0)
        asg = ctx.create_array([n], "i32", ctx.dist.row([n], 25_000, devs), 0)
        cen = ctx.create_array([k, d], "i32", ctx.dist.replicated([k, d], devs), 0)
        sums = ctx.create_array([k, d], "i64", ctx.dist.replicated([k, d], devs), 0)
        cnts = ctx.create_array([k], "i64", ctx.dist.replicated([k], devs), 0)
        ctx.launch("ipattern2d_i32", [n, d], [64, 16], ctx.dist.block_work([n, d], [64, 16], [25_024, d], devs), [n, d, mod, Arr(pts)],
                   "global [i, j] => write out[i,j]")
        wk = ctx.dist.block_work([k, d], [16, 16], [k, d], devs)
        ctx.launch("ipattern2d_i32", [k, d], [16, 16], wk, [k, d, mod - 3, Arr(cen)], "global [i, j] => write out[i,j]")
        w1 = ctx.dist.block_work([n], [64], [25_024], devs)
        for _ in range(2):
            ctx.launch("kmeans_assign_i32", [n], [64], w1, [n, k, d, Arr(asg), Arr(pts), Arr(cen)],
                       "global i => write assign[i], read points[i,:], read centroids[:,:]")
            ctx.launch("kmeans_update_i32", [n], [64], w1, [n, d, Arr(pts), Arr(asg), Arr(sums), Arr(cnts)],
                       "global i => read points[i,:], read assign[i], reduce(+) sums[:,:], reduce(+) counts[:]")
            ctx.launch("kmeans_finalize_i32", [k, d], [16, 16], wk, [k, d, Arr(cen), Arr(sums), Arr(cnts)],
                       "global [i, j] => readwrite centroids[i,j], read sums[i,j], read counts[i]")
        g_asg, g_cen, g_sums, g_cnts = ctx.read(asg), ctx.read(cen), ctx.read(sums), ctx.read(cnts)
    p = np.empty((n, d), np.int32)
    okern.oracle_ipattern2d_i32(C.c_int64(n), C.c_int64(d), C.c_int64(mod), p.ctypes.data_as(I32))
    c = np.empty((k, d), np.int32)
    okern.oracle_ipattern2d_i32(C.c_int64(k), C.c_int64(d), C.c_int64(mod - 3), c.ctypes.data_as(I32))
    a = np.empty(n, np.int32)
    s = np.empty((k, d), np.int64)
    m = np.empty(k, np.int64)
    for _ in range(2):
        okern.oracle_kmeans_assign_i32(C.c_int64(n), C.c_int64(k), C.c_int64(d), p.ctypes.data_as(I32), c.ctypes.data_as(I32), a.ctypes.data_as(I32))
        okern.oracle_kmeans_update_i32(C.c_int64(n), C.c_int64(k), C.c_int64(d), p.ctypes.data_as(I32), a.ctypes.data_as(I32), s.ctypes.data_as(I64),
                                       m.ctypes.data_as(I64))
        okern.oracle_kmeans_finalize_i32(C.c_int64(k), C.c_int64(d), s.ctypes.data_as(I64), m.ctypes.data_as(I64), c.ctypes.data_as(I32))
    assert np.array_equal(g_asg, a)
    assert np.array_equal(g_sums, s)
    assert np.array_equal(g_cnts, m)
    assert np.array_equal(g_cen, c)


def _np_assign(p, c):
    best = np.zeros(len(p), np.int32)
    bd = np.full(len(p), np.iinfo(np.int64).max, np.int64)
    for j in range(len(c)):
        dd = ((p.astype(np.int64) - c[j].astype(np.int64)) ** 2).sum(axis=1)
        upd = dd < bd  # strict: the first minimum wins (kernels.cpp:283-292)
        bd[upd] = dd[upd]
        best[upd] = j
    return best


@pytest.mark.parametrize("lim,d,k", [(8191, 16, 48), (8191, 5, 48), (1 << 20, 16, 48), (255, 16, 48), (1024, 16, 48), (1025, 16, 48), (4096, 1, 48),
                                     (2, 16, 50), (1, 3, 37), (300, 16, 256)])
def test_kmeans_assign_signed_values(lim, d, k):
    """negative coordinates, |x| at the u32 tier's limit (max distance just below 2^32), a
    padded d < 16, and values past the limit (int64 path); the FP32 tier (sum|x| max|c| <= 2^24:
    lim 255, exactly 2^24 at lim 1024 with d 16, and d 1) and just past its bound (lim 1025);
    ties included (duplicate centroids; lim 1-2: most points tie between many centroids, inside
    and across the centred tier's centroid groups, and k not a multiple of the group size)"""
    rng = np.random.default_rng(7)
    n = 20_011
    p = rng.integers(-lim, lim + 1, size=(n, d), dtype=np.int64).astype(np.int32)
    c = rng.integers(-lim, lim + 1, size=(k, d), dtype=np.int64).astype(np.int32)
    c[7] = c[3]
    p[:4] = lim
    c[0] = -lim
    with mb.context(workers=1, devices=1, num_gpus=1) as ctx:
        dv = ctx.devices
        pts = ctx.create_array([n, d], "i32", ctx.dist.single([n, d], dv[0]), 0)
        asg = ctx.create_array([n], "i32", ctx.dist.single([n], dv[0]), 0)
        cen = ctx.create_array([k, d], "i32", ctx.dist.single([k, d], dv[0]), 0)
        ctx.write(pts, p)
        ctx.write(cen, c)
        ctx.launch("kmeans_assign_i32", [n], [128], ctx.dist.block_work([n], [128], [-(-n // 128) * 128], dv), [n, k, d, Arr(asg), Arr(pts), Arr(cen)],
                   "global i => write assign[i], read points[i,:], read centroids[:,:]")
        got = ctx.read(asg)
    assert np.array_equal(got, _np_assign(p, c))


@pytest.mark.parametrize("d", [16, 3])
def test_kmeans_update_full_range_values(d):
    """full-range int32 coordinates: the per-CTA signed i32 sums overflow constantly, so the
    wrap counters must carry the exact int64 total"""
    rng = np.random.default_rng(11)
    n, k = 300_007, 40
    p = rng.integers(-(1 << 31), 1 << 31, size=(n, d), dtype=np.int64).astype(np.int32)
    p[: n // 2] = np.abs(p[: n // 2].astype(np.int64)).clip(0, (1 << 31) - 1).astype(np.int32)  # long positive runs
    a = rng.integers(0, k, size=n, dtype=np.int32)
    a[:1000] = 5
    with mb.context(workers=1, devices=2, num_gpus=1) as ctx:
        dv = ctx.devices
        half = (n + 1) // 2
        pts = ctx.create_array([n, d], "i32", ctx.dist.row([n, d], half, dv), 0)
        asg = ctx.create_array([n], "i32", ctx.dist.row([n], half, dv), 0)
        sums = ctx.create_array([k, d], "i64", ctx.dist.replicated([k, d], dv), 0)
        cnts = ctx.create_array([k], "i64", ctx.dist.replicated([k], dv), 0)
        ctx.write(pts, p)
        ctx.write(asg, a)
        ctx.launch("kmeans_update_i32", [n], [128], ctx.dist.block_work([n], [128], [-(-half // 128) * 128], dv), [n, d, Arr(pts), Arr(asg), Arr(sums), Arr(cnts)],
                   "global i => read points[i,:], read assign[i], reduce(+) sums[:,:], reduce(+) counts[:]")
        g_s, g_c = ctx.read(sums), ctx.read(cnts)
    want_s = np.zeros((k, d), np.int64)
    np.add.at(want_s, a, p.astype(np.int64))
    assert np.array_equal(g_c, np.bincount(a, minlength=k))
    assert np.array_equal(g_s, want_s)
