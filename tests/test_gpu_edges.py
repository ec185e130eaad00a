"""Edge cases and BASELINE-size properties for the C1/C2/C4 kernels.

* heat2d on ragged grids (1x1, single rows/columns, widths that are not a multiple of the
  128-bit vector, column-split tiles whose chunks start at unaligned columns, 2D halos) with
  random inputs: bit-exact against the C oracle (oracle/oracle.c, pinned to the reference in
  tests/test_oracle.py).
* heat2d at the C2 size (65536^2, 4 logical devices on the GPU): one distributed step, rows
  around every chunk boundary and both domain edges checked bit-exact against the oracle's
  band restatement (oracle_heat2d_rows) on inputs restated on the host.
* histogram at n = 1e9 (65536 bins) against the oracle exactly, and the C4 size n = 4e9
  through the total count.
* int32 k-means at the C4 size (n = 1e9, d = 16, k = 256): sampled assignments against an exact
  int64 host argmin (first minimum), every point counted once, and the per-dimension sums equal
  to the closed form of the input pattern.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr

pytestmark = pytest.mark.gpu
HEAT = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"
F32 = C.POINTER(C.c_float)


def oracle_heat(okern, a, iters, alpha=0.1):
    rows, cols = a.shape
    cur = np.ascontiguousarray(a, dtype=np.float32).copy()
    nxt = np.empty_like(cur)
    for _ in range(iters):
        okern.oracle_heat2d(C.c_int64(rows), C.c_int64(cols), C.c_double(alpha), cur.ctypes.data_as(F32), nxt.ctypes.data_as(F32))
        cur, nxt = nxt, cur
    return cur


CASES = [
    # rows, cols, chunk extents, halo, devices, block
    (1, 1, (1, 1), (1, 1), 1, (1, 1)),
    (1, 7, (1, 7), (1, 1), 1, (1, 4)),
    (7, 1, (4, 1), (1, 0), 2, (2, 1)),
    (3, 1030, (3, 1030), (1, 1), 1, (3, 16)),
    (129, 1027, (33, 1027), (1, 0), 4, (3, 13)),
    (64, 96, (32, 48), (1, 1), 4, (8, 8)),
    (50, 301, (50, 101), (0, 1), 3, (5, 7)),
    (257, 515, (65, 259), (1, 1), 4, (13, 37)),
]


@pytest.mark.parametrize("rows,cols,ext,halo,ndev,block", CASES)
def test_heat2d_ragged_shapes(okern, rows, cols, ext, halo, ndev, block):
    x = np.random.default_rng(rows * 1000 + cols).standard_normal((rows, cols)).astype(np.float32)
    iters = 3
    with mb.context(workers=1, devices=ndev, num_gpus=1) as ctx:
        devs = ctx.devices
        dist = lambda: ctx.dist.stencil([rows, cols], list(ext), list(halo), devs)  # noqa: E731
        a = ctx.create_array([rows, cols], "f32", dist(), 0)
        b = ctx.create_array([rows, cols], "f32", dist(), 0)
        ctx.write(a, x)
        sb = [-(-e // bl) * bl for e, bl in zip(ext, block)]  # superblocks: whole blocks covering a chunk
        work = ctx.dist.block_work([rows, cols], list(block), sb, devs)
        for _ in range(iters):
            ctx.launch("heat2d", [rows, cols], list(block), work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
            a, b = b, a
        got = ctx.read(a)
        assert ctx.replicas_coherent(a)
    want = oracle_heat(okern, x, iters)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def ramp_rows(r0, r1, cols, mod=1000):
    """ramp2d_f32 (oracle_ramp2d_f32) for rows [r0, r1), restated in numpy (same IEEE ops)"""
    i = np.arange(r0, r1, dtype=np.int64)[:, None]
    j = np.arange(cols, dtype=np.int64)[None, :]
    return (0.0 + (1.0 * ((i * 31 + j * 17 + 7) % mod).astype(np.float64)) / float(mod)).astype(np.float32)


def test_heat2d_full_size_bands(okern):
    rows = cols = 65536
    parts = 4
    with mb.context(workers=1, devices=parts, num_gpus=1) as ctx:
        devs = ctx.devices
        dist = lambda: ctx.dist.stencil([rows, cols], [rows // parts, cols], [1, 0], devs)  # noqa: E731
        a = ctx.create_array([rows, cols], "f32", dist(), 0)
        b = ctx.create_array([rows, cols], "f32", dist(), 0)
        work = ctx.dist.block_work([rows, cols], [16, 16], [rows // parts, cols], devs)
        ctx.launch("ramp2d_f32", [rows, cols], [16, 16], work, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
        ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
        got = ctx.read(b)
        assert ctx.replicas_coherent(b)
    bands = [(0, 3)] + [(k * rows // parts - 2, k * rows // parts + 2) for k in range(1, parts)] + [(rows - 3, rows), (31337, 31342)]
    for r0, r1 in bands:
        lo, hi = max(0, r0 - 1), min(rows, r1 + 1)
        src = np.ascontiguousarray(ramp_rows(lo, hi, cols))
        want = np.empty((r1 - r0, cols), np.float32)
        okern.oracle_heat2d_rows(C.c_int64(rows), C.c_int64(cols), C.c_double(0.1), src.ctypes.data_as(F32), C.c_int64(lo), C.c_int64(hi - lo),
                                 want.ctypes.data_as(F32), C.c_int64(r0), C.c_int64(r1))
        assert np.array_equal(got[r0:r1].view(np.uint32), want.view(np.uint32)), (r0, r1)


def _histogram(n, bins, seed=12345):
    with mb.context(workers=1, devices=1, num_gpus=1) as ctx:
        dv = ctx.devices
        x = ctx.create_array([n], "i32", ctx.dist.single([n], dv[0]), 0)
        h = ctx.create_array([bins], "i64", ctx.dist.single([bins], dv[0]), 0)
        w = ctx.dist.block_work([n], [256], [n], dv)
        ctx.launch("hpattern1d", [n], [256], w, [n, bins, seed, Arr(x)], "global i => write out[i]")
        ctx.launch("histogram", [n], [256], w, [n, bins, Arr(x), Arr(h)], "global i => read x[i], reduce(+) hist[:]")
        return ctx.read(h)


def test_histogram_1e9_matches_oracle(okern):
    n, bins = 1_000_000_000, 65536
    got = _histogram(n, bins)
    want = np.empty(bins, np.int64)
    okern.oracle_histogram_hashed(C.c_int64(0), C.c_int64(n), C.c_int64(bins), C.c_int64(12345), want.ctypes.data_as(C.POINTER(C.c_int64)))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("bins", [256, 65536])
def test_histogram_c4_size_counts_every_element(bins):
    n = 4_000_000_000
    got = _histogram(n, bins)
    assert int(got.sum()) == n and (got >= 0).all()


def test_kmeans_c4_size_properties():
    n, k, d = 1_000_000_000, 256, 16
    with mb.context(workers=1, devices=1, num_gpus=1) as ctx:
        dv = ctx.devices
        pts = ctx.create_array([n, d], "i32", ctx.dist.single([n, d], dv[0]), 0)
        asg = ctx.create_array([n], "i32", ctx.dist.single([n], dv[0]), 0)
        cen = ctx.create_array([k, d], "i32", ctx.dist.single([k, d], dv[0]), 0)
        sums = ctx.create_array([k, d], "i64", ctx.dist.single([k, d], dv[0]), 0)
        cnts = ctx.create_array([k], "i64", ctx.dist.single([k], dv[0]), 0)
        ctx.launch("ipattern2d_i32", [n, d], [256, 16], ctx.dist.block_work([n, d], [256, 16], [n, d], dv), [n, d, 1000, Arr(pts)],
                   "global [i, j] => write out[i,j]")
        ctx.launch("ipattern2d_i32", [k, d], [16, 16], ctx.dist.block_work([k, d], [16, 16], [k, d], dv), [k, d, 997, Arr(cen)],
                   "global [i, j] => write out[i,j]")
        w = ctx.dist.block_work([n], [256], [n], dv)
        ctx.launch("kmeans_assign_i32", [n], [256], w, [n, k, d, Arr(asg), Arr(pts), Arr(cen)],
                   "global i => write assign[i], read points[i,:], read centroids[:,:]")
        ctx.launch("kmeans_update_i32", [n], [256], w, [n, d, Arr(pts), Arr(asg), Arr(sums), Arr(cnts)],
                   "global i => read points[i,:], read assign[i], reduce(+) sums[:,:], reduce(+) counts[:]")
        a = ctx.read(asg)
        s = ctx.read(sums)
        c = ctx.read(cnts)
        centroids = ctx.read(cen).astype(np.int64)
    assert int(c.sum()) == n
    # (31 i + 17 j + 7) mod 1000 runs through a permutation of 0..999 every 1000 rows
    assert (s.sum(axis=0) == (n // 1000) * 499500).all()
    idx = np.random.default_rng(5).integers(0, n, 4096)
    j = np.arange(d, dtype=np.int64)
    p = (idx[:, None] * 31 + j[None, :] * 17 + 7) % 1000
    dist = ((p[:, None, :] - centroids[None, :, :]) ** 2).sum(axis=2)
    assert np.array_equal(a[idx], dist.argmin(axis=1).astype(np.int32))  # argmin: first minimum, like the reference
    # the counts agree with the assignment vector
    assert np.array_equal(np.bincount(a, minlength=k), c)


def test_heat2d_random_layouts(okern):
    """random grids, chunkings (row and column splits, halos), block shapes and alphas: the
    TMA-staged kernel, its scalar tail and the register kernel where the TMA one does not apply
    must all agree with the oracle bit for bit"""
    rng = np.random.default_rng(2024)
    for case in range(30):
        rows = int(rng.integers(1, 700))
        cols = int(rng.integers(1, 1300))
        ndev = int(rng.integers(1, 5))
        er = int(rng.integers(1, rows + 1))
        ec = cols if rng.random() < 0.6 else int(rng.integers(1, cols + 1))
        halo = [1, 1 if ec < cols else int(rng.integers(0, 2))]
        block = [int(rng.integers(1, 33)), int(rng.integers(1, 65))]
        alpha = float(rng.choice([0.1, 0.25, 0.01]))
        iters = int(rng.integers(1, 4))
        x = rng.standard_normal((rows, cols)).astype(np.float32)
        with mb.context(workers=1, devices=ndev, num_gpus=1) as ctx:
            devs = ctx.devices
            dist = lambda: ctx.dist.stencil([rows, cols], [er, ec], halo, devs)  # noqa: E731
            a = ctx.create_array([rows, cols], "f32", dist(), 0)
            b = ctx.create_array([rows, cols], "f32", dist(), 0)
            ctx.write(a, x)
            sb = [-(-er // block[0]) * block[0], -(-ec // block[1]) * block[1]]
            work = ctx.dist.block_work([rows, cols], block, sb, devs)
            for _ in range(iters):
                ctx.launch("heat2d", [rows, cols], block, work, [rows, cols, alpha, Arr(b), Arr(a)], HEAT)
                a, b = b, a
            got = ctx.read(a)
        want = oracle_heat(okern, x, iters, alpha)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (case, rows, cols, er, ec, halo, block)


def _heat_full(parts, steps):
    rows = cols = 65536
    with mb.context(workers=1, devices=parts, num_gpus=1, retain_plan=False) as ctx:
        devs = ctx.devices
        dist = lambda: ctx.dist.stencil([rows, cols], [rows // parts, cols], [1, 0], devs)  # noqa: E731
        a = ctx.create_array([rows, cols], "f32", dist(), 0)
        b = ctx.create_array([rows, cols], "f32", dist(), 0)
        work = ctx.dist.block_work([rows, cols], [16, 16], [rows // parts, cols], devs)
        ctx.launch("ramp2d_f32", [rows, cols], [16, 16], work, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
        ctx.launch_repeat("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT, steps, swap=(a, b))
        out = b if steps % 2 else a
        got = ctx.read(out)
        assert ctx.replicas_coherent(out)
    return got


def test_heat2d_full_size_multi_step(okern):
    """BASELINE C2 at full size, several steps: the 4-device run equals the 1-device run bit for
    bit over all 65536^2 cells (distributed == serial, test_runtime.cpp:67-72), and bands at the
    chunk boundaries, the domain edges and the middle equal the C oracle, which evolves each band
    from the ramp with `steps` extra rows on either side (the dependency cone of the stencil)"""
    rows = cols = 65536
    steps = 5
    got = _heat_full(4, steps)
    serial = _heat_full(1, steps)
    assert np.array_equal(got.view(np.uint32), serial.view(np.uint32))
    del serial
    bands = [(0, 8)] + [(k * rows // 4 - 4, k * rows // 4 + 4) for k in range(1, 4)] + [(rows - 8, rows), (40000, 40008)]
    for r0, r1 in bands:
        lo, hi = max(0, r0 - steps), min(rows, r1 + steps)
        cur = np.ascontiguousarray(ramp_rows(lo, hi, cols))
        for _ in range(steps):
            nlo = lo if lo == 0 else lo + 1
            nhi = hi if hi == rows else hi - 1
            nxt = np.empty((nhi - nlo, cols), np.float32)
            okern.oracle_heat2d_rows(C.c_int64(rows), C.c_int64(cols), C.c_double(0.1), cur.ctypes.data_as(F32), C.c_int64(lo), C.c_int64(hi - lo),
                                     nxt.ctypes.data_as(F32), C.c_int64(nlo), C.c_int64(nhi))
            cur, lo, hi = nxt, nlo, nhi
        assert np.array_equal(got[r0:r1].view(np.uint32), cur[r0 - lo:r1 - lo].view(np.uint32)), (r0, r1)
