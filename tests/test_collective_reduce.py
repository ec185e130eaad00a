"""Collective reduce trees (cfg.collective_reduce): the reference's send-to-root tree
(planner.cpp:389-517) becomes one allreduce task per worker (NCCL between processes, a
peer-memory combine in one process). Plan structure and serial-order soundness on CPU; on the
GPU the in-process combine must equal the tree bit for bit, float sums included, because it
combines the members in the root reduce's input order."""
import numpy as np
import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr

from test_planner_parity import assert_orders_conflicts

HIST = "global i => read x[i], reduce(+) hist[:]"
ROWRED = "global [i, j] => read A[i,j], reduce(+) sums[i]"


def _hist_plan(ctx, n, bins, work_devs):
    devs = ctx.devices
    x = ctx.create_array([n], "i32", ctx.dist.row([n], n // len(devs), devs), 0)
    h = ctx.create_array([bins], "i64", ctx.dist.replicated([bins], devs), 0)
    w = ctx.dist.block_work([n], [16], [n // len(work_devs)], work_devs)
    ctx.launch("hpattern1d", [n], [16], ctx.dist.block_work([n], [16], [n // len(devs)], devs), [n, bins, 3, Arr(x)], "global i => write out[i]")
    ctx.launch("histogram", [n], [16], w, [n, bins, Arr(x), Arr(h)], HIST)
    return x, h


def test_plan_has_one_allreduce_per_worker():
    with mb.context(workers=3, devices=2, execute=False, collective_reduce=True, record_accesses=True) as ctx:
        devs = ctx.devices
        work = [d for d in devs if d[0] < 2]  # worker 2 has no partial: it joins with an identity box
        _hist_plan(ctx, 1536, 40, work)
        plan = ctx.plan()
        ars = [t for t in plan if t["kind"] == "allreduce"]
        assert [t["worker"] for t in ars] == [0, 1, 2]
        assert len({t["tag"] for t in ars}) == 1
        ids = [t["id"] for t in ars]
        assert ids == list(range(ids[0], ids[0] + 3))  # consecutive: the in-process combine relies on it
        data = ars[0]["inputs"]
        assert all(t["inputs"] == data for t in ars) and len(data) == 2
        assert [ars[0]["output"], ars[1]["output"]] == data
        filler = ars[2]["output"]
        assert filler not in data
        creates = {t["chunk"]: t for t in plan if t["kind"] == "create"}
        assert creates[filler]["fill"] == 3  # identity
        # no send/recv in the reduce tree; each replica gets a local copy from its own worker
        launch_tasks = [t for t in plan if t["id"] > ids[-1]]
        assert not any(t["kind"] in ("send", "recv") for t in launch_tasks)
        copies = [t for t in launch_tasks if t["kind"] == "copy"]
        assert len(copies) == len(devs)
        member = {t["worker"]: t["output"] for t in ars}
        for c in copies:
            assert c["src"] == member[c["worker"]]
        assert_orders_conflicts(ctx, plan)


def test_single_worker_needs_no_collective():
    with mb.context(workers=1, devices=4, execute=False, collective_reduce=True) as ctx:
        _hist_plan(ctx, 1024, 16, ctx.devices)
        assert not any(t["kind"] == "allreduce" for t in ctx.plan())


def test_default_keeps_the_reference_tree():
    with mb.context(workers=2, devices=1, execute=False) as ctx:
        _hist_plan(ctx, 1024, 16, ctx.devices)
        kinds = [t["kind"] for t in ctx.plan()]
        assert "allreduce" not in kinds and "send" in kinds


def _run(collective, fn):
    with mb.context(workers=2, devices=2, num_gpus=1, collective_reduce=collective) as ctx:
        return fn(ctx)


@pytest.mark.gpu
def test_in_process_allreduce_matches_tree_histogram():
    n, bins = 1 << 20, 1000

    def fn(ctx):
        _, h = _hist_plan(ctx, n, bins, ctx.devices)
        return ctx.read(h), ctx.replicas_coherent(h), ctx.exec_stats()

    tree, ok_t, st_t = _run(False, fn)
    coll, ok_c, st_c = _run(True, fn)
    assert ok_t and ok_c
    assert np.array_equal(tree, coll)
    assert st_t["bytes_sent"] > 0 and st_c["bytes_sent"] == 0  # no messages in the collective tree


@pytest.mark.gpu
def test_in_process_allreduce_float_sum_bit_exact():
    rows, cols = 4096, 512

    def fn(ctx):
        devs = ctx.devices
        a = ctx.create_array([rows, cols], "f32", ctx.dist.col([rows, cols], cols // 4, devs), 0)
        s = ctx.create_array([rows], "f32", ctx.dist.replicated([rows], devs), 0)
        rng = np.random.default_rng(5)
        ctx.write(a, rng.standard_normal((rows, cols)).astype(np.float32) * 1e3)
        w = ctx.dist.block_work([rows, cols], [16, 16], [rows, cols // 4], devs)  # each superblock: a column slab of every row
        for _ in range(3):
            ctx.launch("row_reduce", [rows, cols], [16, 16], w, [rows, cols, Arr(a), Arr(s)], ROWRED)
        return ctx.read(s)

    tree = _run(False, fn)
    coll = _run(True, fn)
    assert np.array_equal(tree.view(np.uint32), coll.view(np.uint32))


@pytest.mark.gpu
def test_in_process_allreduce_with_identity_member():
    """worker 1 has no partial and joins with an identity box"""
    n = 4096

    def fn(ctx):
        devs = ctx.devices
        x = ctx.create_array([n], "i32", ctx.dist.row([n], n // 4, devs), 0)
        h = ctx.create_array([64], "i64", ctx.dist.replicated([64], devs), 0)
        ctx.launch("hpattern1d", [n], [16], ctx.dist.block_work([n], [16], [n // 4], devs), [n, 64, 9, Arr(x)], "global i => write out[i]")
        work = [d for d in devs if d[0] == 0]
        ctx.launch("histogram", [n], [16], ctx.dist.block_work([n], [16], [n // 2], work), [n, 64, Arr(x), Arr(h)], HIST)
        return ctx.read(h)

    assert np.array_equal(_run(False, fn), _run(True, fn))
