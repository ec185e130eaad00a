"""Asynchronous host transfers (mt_array_write_async / mt_array_read_async): planned as
host_write / host_read tasks, so launches are ordered after the upload that feeds them and
the download after the launch that produces the result. CPU: plan structure (a read covers
the domain exactly once, dependencies order it). GPU: pipelined steps over two array sets
equal the synchronous path bit for bit."""
import numpy as np
import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr

from test_planner_parity import assert_orders_conflicts, closure

HEAT = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"


def _vol(box):
    lo, hi = box
    v = 1
    for a, b in zip(lo, hi):
        v *= b - a
    return v


def test_host_tasks_cover_and_order():
    rows, cols = 512, 64
    with mb.context(workers=2, devices=2, execute=False, record_accesses=True) as ctx:
        devs = ctx.devices
        d = ctx.dist.stencil([rows, cols], [rows // 4, cols], [1, 0], devs)
        a = ctx.create_array([rows, cols], "f32", d, 0)
        b = ctx.create_array([rows, cols], "f32", d, 0)
        w = ctx.dist.block_work([rows, cols], [16, 16], [rows // 4, cols], devs)
        first = ctx.plan_size()
        ctx.lib.check(ctx.lib.array_write_async(ctx.h, a, 0x1000, rows * cols * 4))  # plan-only: the address is never used
        ctx.launch("heat2d", [rows, cols], [16, 16], w, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
        ctx.lib.check(ctx.lib.array_read_async(ctx.h, b, 0x2000, rows * cols * 4))
        plan = ctx.plan()
        writes = [t for t in plan if t["kind"] == "host_write"]
        reads = [t for t in plan if t["kind"] == "host_read"]
        assert len(writes) == 4 and all(t["host"] == 0x1000 for t in writes)
        # every chunk written whole (halo rows included)
        assert sorted(_vol(t["region"]) for t in writes) == sorted(_vol((c.lo, c.hi)) for c in ctx.chunks(a))
        # the read covers the domain exactly once
        assert sum(_vol(t["region"]) for t in reads) == rows * cols
        reach = closure(plan)
        execs = [t for t in plan if t["kind"] == "execute" and t["id"] >= first]
        for e in execs:
            assert any(w_["id"] in reach[e["id"]] for w_ in writes)
        for r in reads:
            assert any(e["id"] in reach[r["id"]] for e in execs)
        assert_orders_conflicts(ctx, plan)


@pytest.mark.gpu
def test_pipelined_host_io_matches_synchronous():
    import torch
    rows, cols, iters, steps = 1024, 2048, 6, 4
    rng = np.random.default_rng(3)
    inputs = [rng.standard_normal((rows, cols)).astype(np.float32) for _ in range(steps)]

    def arrays(ctx):
        devs = ctx.devices
        d = lambda: ctx.dist.stencil([rows, cols], [rows // 2, cols], [1, 0], devs)  # noqa: E731
        return ctx.create_array([rows, cols], "f32", d(), 0), ctx.create_array([rows, cols], "f32", d(), 0)

    def run(ctx, a, b, w):
        for _ in range(iters):
            ctx.launch("heat2d", [rows, cols], [16, 16], w, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
            a, b = b, a
        return a

    want = []
    with mb.context(workers=1, devices=2, num_gpus=1) as ctx:
        a, b = arrays(ctx)
        w = ctx.dist.block_work([rows, cols], [16, 16], [rows // 2, cols], ctx.devices)
        for x in inputs:
            ctx.write(a, x)
            want.append(ctx.read(run(ctx, a, b, w)))
    with mb.context(workers=1, devices=2, num_gpus=1) as ctx:
        sets = [arrays(ctx), arrays(ctx)]
        w = ctx.dist.block_work([rows, cols], [16, 16], [rows // 2, cols], ctx.devices)
        host_in = [torch.from_numpy(x).pin_memory() for x in inputs]
        host_out = [torch.empty((rows, cols), dtype=torch.float32).pin_memory() for _ in range(steps)]
        for s in range(steps):
            a, b = sets[s % 2]
            ctx.write_async(a, host_in[s])
            ctx.read_async(run(ctx, a, b, w), host_out[s])
        ctx.synchronize()
        st = ctx.exec_stats()
        got = [t.numpy() for t in host_out]
    for g, x in zip(got, want):
        assert np.array_equal(g.view(np.uint32), x.view(np.uint32))
    assert st["host_read_bytes"] == steps * rows * cols * 4


def test_box_transfers_plan_the_same_tasks():
    """the host box changes only the host side of each task (src_region), never the task
    sequence, so ranks passing different boxes keep identical plans; bad boxes are rejected"""
    rows, cols = 256, 64

    def plan(box):
        with mb.context(workers=2, devices=1, execute=False) as ctx:
            devs = ctx.devices
            d = ctx.dist.stencil([rows, cols], [rows // 2, cols], [1, 0], devs)
            a = ctx.create_array([rows, cols], "f32", d, 0)
            r = mb._capi.Rect.make(*box) if box else None
            vol = rows * cols if box is None else _vol(box) * 1
            if box is None:
                ctx.lib.check(ctx.lib.array_write_async(ctx.h, a, 0x1000, vol * 4))
                ctx.lib.check(ctx.lib.array_read_async(ctx.h, a, 0x1000, vol * 4))
            else:
                ctx.lib.check(ctx.lib.array_write_box_async(ctx.h, a, r, 0x1000, vol * 4))
                ctx.lib.check(ctx.lib.array_read_box_async(ctx.h, a, r, 0x1000, vol * 4))
            return [{k: v for k, v in t.items() if k != "host_box"} for t in ctx.plan()], [t.get("host_box") for t in ctx.plan()]

    base, _ = plan(None)
    for box in [((0, 0), (129, 64)), ((127, 0), (256, 64))]:
        tasks, boxes = plan(box)
        assert tasks == base
        assert all(b == box for b in boxes if b is not None)
    with mb.context(workers=1, devices=1, execute=False) as ctx:
        a = ctx.create_array([rows, cols], "f32", ctx.dist.single([rows, cols], ctx.devices[0]), 0)
        with pytest.raises(mb.ValidationError):
            ctx.lib.check(ctx.lib.array_write_box_async(ctx.h, a, mb._capi.Rect.make((0, 0), (rows + 1, cols)), 0x1000, (rows + 1) * cols * 4))
        with pytest.raises(mb.ValidationError):
            ctx.lib.check(ctx.lib.array_write_box_async(ctx.h, a, mb._capi.Rect.make((0, 0), (8, cols)), 0x1000, 8 * cols * 4 - 4))
