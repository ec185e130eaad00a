"""Known answers of the reference's own unit suites (proj/tests/unit), asked of this planner
through its Python / C-ABI surface. The plan-parity tests compare whole plans with the live
reference; these restate the hand-derived values the reference pins, so a reader can match
them line by line."""
import os
import sys

import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr

sys.path.insert(0, os.path.dirname(__file__))
from test_acceptance_plan import _planned_regions  # noqa: E402


def devices(workers, per):
    return mb.context(workers=workers, devices=per, execute=False).devices


def test_block_distribution_of_one_million_threads():
    """test_distribution.cpp:24-34"""
    devs = devices(2, 2)
    ctx = mb.context(workers=2, devices=2, execute=False)
    w = ctx.dist.block_work([1000000], [16], [64000], devs)
    assert len(w) == 16
    assert [s.device for s in w] == [tuple(devs[s % 4]) for s in range(16)]
    assert (w[0].lo, w[0].hi) == ((0,), (4000,))
    assert (w[15].lo, w[15].hi) == ((60000,), (62500,))  # ragged last superblock


def test_stencil_distribution_halo_and_overlap():
    """test_distribution.cpp:89-104"""
    ctx = mb.context(workers=2, devices=2, execute=False)
    d = ctx.dist.stencil([1000000], [64000], [1], ctx.devices)
    assert len(d) == 16
    assert (d[0].lo, d[0].hi) == ((0,), (64001,))
    assert (d[1].lo, d[1].hi) == ((63999,), (128001,))
    assert (d[15].lo, d[15].hi) == ((959999,), (1000000,))
    for a, b in zip(d, d[1:]):
        assert min(a.hi[0], b.hi[0]) - max(a.lo[0], b.lo[0]) == 2  # neighbours share twice the halo


def test_tile_distribution_of_a_12x12_array():
    """test_distribution.cpp:84-87"""
    ctx = mb.context(workers=1, devices=4, execute=False)
    assert len(ctx.dist.tile([12, 12], [6, 6], ctx.devices)) == 4


def test_stencil_regions_interior_and_clipped():
    """test_annotation.cpp:105-126: interior superblock [63999, 128001) / [64000, 128000), and the
    left halo clipped at the domain edge, [0, 64001)"""
    text = "global i => read A[i-1:i+1], read B[i]"
    got = _planned_regions(text, [1000000], [16], ([64000], [128000]), [[1000000], [1000000]])
    assert got == [((63999,), (128001,)), ((64000,), (128000,))]
    got = _planned_regions(text, [1000000], [16], ([0], [64000]), [[1000000], [1000000]])
    assert got[0] == ((0,), (64001,))


def test_matmul_regions_for_a_corner_superblock():
    """test_annotation.cpp:128-141"""
    text = "global [i, j] => read A[i,:], read B[:,j], read C[i,j]"
    got = _planned_regions(text, [8, 8], [2, 2], ([0, 0], [4, 4]), [[8, 8], [8, 8], [8, 8]])
    assert got == [((0, 0), (4, 8)), ((0, 0), (8, 4)), ((0, 0), (4, 4))]


@pytest.mark.parametrize("compat", [True, False])
def test_stencil_launch_task_counts(compat):
    """test_planner.cpp:74-101: 4 executes, no temporaries, 4 propagation copies, 2 send/recv"""
    ctx = mb.context(workers=2, devices=2, execute=False, compat_deps=compat)
    n = 256000
    dist = lambda: ctx.dist.stencil([n], [64000], [1], ctx.devices)  # noqa: E731
    a = ctx.create_array([n], "f32", dist(), 1)
    b = ctx.create_array([n], "f32", dist(), 0)
    first, last = ctx.launch("stencil1d", [n], [16], ctx.dist.block_work([n], [16], [64000], ctx.devices), [n, Arr(b), Arr(a)],
                             "global i => read input[i-1:i+1], write output[i]")
    kinds = [t["kind"] for t in ctx.plan(first, last)]
    assert {k: kinds.count(k) for k in set(kinds)} == {"execute": 4, "copy": 4, "send": 2, "recv": 2}


def test_replicated_vectors_need_no_assembly():
    """test_planner.cpp:196-223: x[:] reads bind to each device's replica (no temporaries); y's
    writes only propagate to the other replicas"""
    ctx = mb.context(workers=2, devices=2, execute=False)
    rows, devs = 64, ctx.devices
    y = ctx.create_array([rows], "f32", ctx.dist.replicated([rows], devs), 0)
    vals = ctx.create_array([rows, 8], "f32", ctx.dist.row([rows, 8], 16, devs), 1)
    cols = ctx.create_array([rows, 8], "i64", ctx.dist.row([rows, 8], 16, devs), 0)
    x = ctx.create_array([rows], "f32", ctx.dist.replicated([rows], devs), 1)
    first, last = ctx.launch("spmv_ell", [rows], [4], ctx.dist.block_work([rows], [4], [16], devs), [rows, 8, Arr(y), Arr(vals), Arr(cols), Arr(x)],
                             "global i => write y[i], read vals[i,:], read cols[i,:], read x[:]")
    plan = ctx.plan(first, last)
    assert not [t for t in plan if t["kind"] == "create"]
    for t in plan:
        if t["kind"] == "copy":
            assert not ctx.chunk_meta(t["src"])[2]


def test_column_sum_reduction_hierarchy():
    """test_planner.cpp:225-250: 2 partials + 1 worker output + 1 final output, 2 combines,
    4 deletes, 1 write-back copy"""
    ctx = mb.context(workers=1, devices=2, execute=False)
    devs = ctx.devices
    a = ctx.create_array([8, 8], "f32", ctx.dist.col([8, 8], 4, devs), 1)
    s = ctx.create_array([8], "f32", ctx.dist.single([8], devs[0]), 0)
    w = ctx.dist.block_work([8, 8], [2, 2], [8, 4], devs)
    assert len(w) == 2
    first, last = ctx.launch("row_reduce", [8, 8], [2, 2], w, [8, 8, Arr(a), Arr(s)], "global [i, j] => read A[i,j], reduce(+) sums[i]")
    kinds = [t["kind"] for t in ctx.plan(first, last)]
    assert (kinds.count("create"), kinds.count("reduce"), kinds.count("delete"), kinds.count("copy")) == (4, 2, 4, 1)


def test_single_superblock_reduction():
    """test_planner.cpp:252-266"""
    ctx = mb.context(workers=1, devices=1, execute=False)
    d = ctx.devices[0]
    a = ctx.create_array([8, 8], "f32", ctx.dist.single([8, 8], d), 1)
    s = ctx.create_array([8], "f32", ctx.dist.single([8], d), 0)
    first, last = ctx.launch("row_reduce", [8, 8], [2, 2], ctx.dist.block_work([8, 8], [2, 2], [8, 8], [d]), [8, 8, Arr(a), Arr(s)],
                             "global [i, j] => read A[i,j], reduce(+) sums[i]")
    kinds = [t["kind"] for t in ctx.plan(first, last)]
    assert (kinds.count("reduce"), kinds.count("create")) == (1, 2)
