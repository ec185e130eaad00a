"""Pinned-host spill tier (executor.cu, spill section): device capacity capped below the
working set; results must stay bit-exact and the bytes moved must stay near the minimum
(the reference's LRU + unconditional write-back moves 2.0-2.4x)."""
import ctypes as C

import numpy as np
import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr

pytestmark = pytest.mark.gpu
HEAT = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"
F = C.POINTER(C.c_float)


def oracle_heat(okern, rows, cols, iters):
    cur = np.empty((rows, cols), np.float32)
    okern.oracle_ramp2d_f32(C.c_int64(rows), C.c_int64(cols), C.c_int64(1000), C.c_double(0.0), C.c_double(1.0), cur.ctypes.data_as(F))
    nxt = np.empty_like(cur)
    for _ in range(iters):
        okern.oracle_heat2d(C.c_int64(rows), C.c_int64(cols), C.c_double(0.1), cur.ctypes.data_as(F), nxt.ctypes.data_as(F))
        cur, nxt = nxt, cur
    return cur


def run_heat(rows, cols, chunk_rows, iters, capacity, lookahead=0):
    with mb.context(workers=1, devices=1, num_gpus=1, device_capacity=capacity, host_capacity=1 << 34, lookahead_tasks=lookahead) as ctx:
        devs = ctx.devices
        dist = lambda: ctx.dist.stencil([rows, cols], [chunk_rows, cols], [1, 0], devs)  # noqa: E731
        a = ctx.create_array([rows, cols], "f32", dist(), 0)
        b = ctx.create_array([rows, cols], "f32", dist(), 0)
        work = ctx.dist.block_work([rows, cols], [16, 16], [chunk_rows, cols], devs)
        ctx.launch("ramp2d_f32", [rows, cols], [16, 16], work, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
        ctx.flush()
        for _ in range(iters):
            ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
            ctx.flush()
            a, b = b, a
        ctx.synchronize()
        stats = ctx.exec_stats()
        out = ctx.read(a)
        coherent = ctx.replicas_coherent(a)
    return out, coherent, stats


def test_spilled_heat2d_is_bit_exact(okern):
    rows, cols, iters = 1024, 4096, 8
    ws = 2 * rows * cols * 4  # 32 MiB working set
    out, coherent, stats = run_heat(rows, cols, 64, iters, capacity=ws // 2)
    assert coherent
    assert stats["evictions"] > 0
    assert stats["peak_device_bytes"] <= ws // 2
    assert np.array_equal(out.view(np.uint32), oracle_heat(okern, rows, cols, iters).view(np.uint32))


def test_spill_traffic_near_minimum():
    """Capacity = 1/2 of the working set. The minimum per iteration is about
    (working set - capacity) each way; Belady over the lookahead plus dirty tracking must
    stay well under the reference LRU's 2.0-2.4x."""
    rows, cols, iters = 2048, 4096, 10
    ws = 2 * rows * cols * 4
    cap = ws // 2
    _, _, stats = run_heat(rows, cols, 128, iters, capacity=cap)
    per_iter_h2d = stats["spill_bytes_h2d"] / iters
    per_iter_d2h = stats["spill_bytes_d2h"] / iters
    minimum = ws - cap
    assert per_iter_h2d <= 1.5 * minimum, (per_iter_h2d / minimum)
    assert per_iter_d2h <= 1.5 * minimum, (per_iter_d2h / minimum)


def test_stencil1d_eviction_matches_serial():
    """test_runtime.cpp:74-85: the 1D stencil under memory pressure equals the unconstrained run."""
    n = 1 << 18

    def run(capacity, host):
        with mb.context(workers=2, devices=2, num_gpus=1, device_capacity=capacity, host_capacity=host) as ctx:
            devs = ctx.devices
            a = ctx.create_array([n], "f32", ctx.dist.stencil([n], [n // 8], [1], devs), 1)
            b = ctx.create_array([n], "f32", ctx.dist.stencil([n], [n // 8], [1], devs), 0)
            w = ctx.dist.block_work([n], [16], [n // 8], devs)
            for _ in range(6):
                ctx.launch("stencil1d", [n], [16], w, [n, Arr(b), Arr(a)], "global i => read input[i-1:i+1], write output[i]")
                ctx.flush()
                a, b = b, a
            return ctx.read(a), ctx.exec_stats()

    free, _ = run(0, 0)
    tight, st = run(n * 4 // 2, 1 << 30)
    assert st["evictions"] > 0
    assert np.array_equal(free.view(np.uint32), tight.view(np.uint32))


def test_disk_tier_below_the_host_tier(okern, tmp_path):
    """device capacity 1/4 of the working set and a host tier of one chunk pair: evicted copies
    must move on to the spill file (memory.cpp:113-159) and come back bit-exact"""
    rows, cols, chunk_rows, iters = 1024, 2048, 64, 6
    ws = 2 * rows * cols * 4  # 16 MiB in 32 chunks of 512 KiB
    chunk = chunk_rows * cols * 4
    with mb.context(workers=1, devices=1, num_gpus=1, device_capacity=ws // 4, host_capacity=6 * chunk, disk_capacity=ws,
                    spill_dir=str(tmp_path)) as ctx:
        devs = ctx.devices
        dist = lambda: ctx.dist.stencil([rows, cols], [chunk_rows, cols], [1, 0], devs)  # noqa: E731
        a = ctx.create_array([rows, cols], "f32", dist(), 0)
        b = ctx.create_array([rows, cols], "f32", dist(), 0)
        work = ctx.dist.block_work([rows, cols], [16, 16], [chunk_rows, cols], devs)
        ctx.launch("ramp2d_f32", [rows, cols], [16, 16], work, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
        ctx.flush()
        for _ in range(iters):
            ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
            ctx.flush()
            a, b = b, a
        ctx.synchronize()
        stats = ctx.exec_stats()
        out = ctx.read(a)
        report = ctx.report_json()
    assert stats["bytes_host_to_disk"] > 0 and stats["bytes_disk_to_host"] > 0
    assert '"bytes_host_to_disk": %d' % stats["bytes_host_to_disk"] in report
    want = oracle_heat(okern, rows, cols, iters)
    assert np.array_equal(out.view(np.uint32), want.view(np.uint32))
    assert list(tmp_path.iterdir()) == []  # the spill file is removed with the context


def test_disk_tier_exhaustion_is_an_execution_error(tmp_path):
    rows, cols, chunk_rows = 1024, 2048, 64
    ws = 2 * rows * cols * 4
    chunk = chunk_rows * cols * 4
    with pytest.raises(mb.ExecutionError):
        with mb.context(workers=1, devices=1, num_gpus=1, device_capacity=ws // 4, host_capacity=4 * chunk, disk_capacity=2 * chunk,
                        spill_dir=str(tmp_path)) as ctx:
            devs = ctx.devices
            dist = lambda: ctx.dist.stencil([rows, cols], [chunk_rows, cols], [1, 0], devs)  # noqa: E731
            a = ctx.create_array([rows, cols], "f32", dist(), 0)
            b = ctx.create_array([rows, cols], "f32", dist(), 0)
            work = ctx.dist.block_work([rows, cols], [16, 16], [chunk_rows, cols], devs)
            ctx.launch("ramp2d_f32", [rows, cols], [16, 16], work, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
            for _ in range(4):
                ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
                a, b = b, a
            ctx.synchronize()
