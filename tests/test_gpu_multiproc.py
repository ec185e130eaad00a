"""One process per worker on the GPU: every rank plans the full plan, executes only its own
worker's tasks, and the cross-worker send/recv tasks (halo rows, reduce partials) move through
the GPU-driven IPC mailbox rings. Two processes share the single test GPU (IPC works within a
device; the spin-waits progress under time-slicing), so this checks correctness, not speed.
The gathered result is compared bit-exact with the single-process run."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
HEAT = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _heat_rank(rank, world, port, rows, cols, iters, q, halo=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    ctx = mb.context(workers=world, devices=1, worker_rank=rank, gpu_base=0)
    ctx.connect_peers()
    devs = ctx.devices
    dist_ = lambda: ctx.dist.stencil([rows, cols], [rows // world, cols], [halo, 0], devs)  # noqa: E731
    a = ctx.create_array([rows, cols], "f32", dist_(), 0)
    b = ctx.create_array([rows, cols], "f32", dist_(), 0)
    work = ctx.dist.block_work([rows, cols], [16, 16], [rows // world, cols], devs)
    ctx.launch("ramp2d_f32", [rows, cols], [16, 16], work, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
    for _ in range(iters):
        ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
        ctx.flush()
        a, b = b, a
    ctx.synchronize()
    out = ctx.read(a)  # local chunks only
    lo = rank * rows // world
    hi = (rank + 1) * rows // world
    q.put((rank, out[lo:hi].copy(), ctx.exec_stats()))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def _two_process_heat(rows, cols, iters, halo=1, world=2):
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_heat_rank, args=(r, world, port, rows, cols, iters, q, halo)) for r in range(world)]
    for p in procs:
        p.start()
    parts = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = np.concatenate([p[1] for p in parts])
    assert all(p[2]["bytes_sent"] > 0 for p in parts)
    with mb.context(workers=1, devices=world, num_gpus=1) as c:
        devs = c.devices
        a = c.create_array([rows, cols], "f32", c.dist.stencil([rows, cols], [rows // world, cols], [halo, 0], devs), 0)
        b = c.create_array([rows, cols], "f32", c.dist.stencil([rows, cols], [rows // world, cols], [halo, 0], devs), 0)
        w = c.dist.block_work([rows, cols], [16, 16], [rows // world, cols], devs)
        c.launch("ramp2d_f32", [rows, cols], [16, 16], w, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
        for _ in range(iters):
            c.launch("heat2d", [rows, cols], [16, 16], w, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
            a, b = b, a
        want = c.read(a)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    return [p[2] for p in parts]


def test_two_process_heat_matches_single_process():
    """10 iterations: each rank sends and receives one halo row per iteration, so the 4-slot ring
    wraps twice; every message is one copy kernel per side, preceded by a one-thread wait kernel
    for every receive and for every send past the ring's 4 slots (exec_stats message_ops)"""
    stats = _two_process_heat(256, 512, 10)
    for st in stats:
        assert st["messages"] == 22  # (ramp + 10 iterations) x (1 send + 1 receive) per rank
        assert st["message_ops"] == 22 + 11 + (11 - 4)


def test_two_process_heat_large_halo_segments():
    """halo [8, 0] rows of 600000 f32 = 19.2 MB per message: larger than one 16 MiB ring slot, so
    the segmented path (stage, per-segment wait / copy / flag) moves them"""
    stats = _two_process_heat(64, 600000, 3, halo=8)
    for st in stats:
        assert st["messages"] == 8  # (ramp + 3 iterations) x (1 send + 1 receive)
        assert st["message_ops"] > st["messages"]


def _hist_rank(rank, world, port, n, bins, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    ctx = mb.context(workers=world, devices=1, worker_rank=rank, gpu_base=0)
    ctx.connect_peers()
    devs = ctx.devices
    per = n // world
    x = ctx.create_array([n], "i32", ctx.dist.row([n], per, devs), 0)
    h = ctx.create_array([bins], "i64", ctx.dist.replicated([bins], devs), 0)
    w = ctx.dist.block_work([n], [128], [per], devs)
    ctx.launch("hpattern1d", [n], [128], w, [n, bins, 5, Arr(x)], "global i => write out[i]")
    ctx.launch("histogram", [n], [128], w, [n, bins, Arr(x), Arr(h)], "global i => read x[i], reduce(+) hist[:]")
    ctx.synchronize()
    q.put((rank, ctx.read(h)))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def test_two_process_reduce_tree(okern):
    """partials travel to the root worker and the result back to every replica via the rings"""
    import ctypes as C
    n, bins, world = 1 << 20, 1000, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_hist_rank, args=(r, world, port, n, bins, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = np.empty(bins, np.int64)
    okern.oracle_histogram_hashed(C.c_int64(0), C.c_int64(n), C.c_int64(bins), C.c_int64(5), want.ctypes.data_as(C.POINTER(C.c_int64)))
    for _, h in res:
        assert np.array_equal(h, want)


def _coll_rank(rank, world, port, n, bins, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    ctx = mb.context(workers=world, devices=1, worker_rank=rank, gpu_base=0, collective_reduce=True)
    try:
        ctx.connect_peers()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", str(e)))
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()
        return
    devs = ctx.devices
    per = n // world
    x = ctx.create_array([n], "i32", ctx.dist.row([n], per, devs), 0)
    h = ctx.create_array([bins], "i64", ctx.dist.replicated([bins], devs), 0)
    w = ctx.dist.block_work([n], [128], [per], devs)
    ctx.launch("hpattern1d", [n], [128], w, [n, bins, 5, Arr(x)], "global i => write out[i]")
    ctx.launch("histogram", [n], [128], w, [n, bins, Arr(x), Arr(h)], "global i => read x[i], reduce(+) hist[:]")
    ctx.synchronize()
    q.put((rank, "ok", ctx.read(h)))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def test_two_process_nccl_allreduce(okern):
    """the reduce tree as ncclAllReduce between processes; NCCL refuses two ranks on one GPU,
    so on a single-GPU box this reports a skip (the in-process combine is covered by
    test_collective_reduce.py, the group ordering across ranks by test_multiproc.py)"""
    import ctypes as C
    n, bins, world = 1 << 20, 1000, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_coll_rank, args=(r, world, port, n, bins, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    errs = [r[2] for r in res if r[1] == "error"]
    if errs:
        import torch
        if torch.cuda.device_count() < world:
            pytest.skip(f"NCCL needs {world} GPUs: {errs[0][:200]}")
        raise AssertionError(errs)
    want = np.empty(bins, np.int64)
    okern.oracle_histogram_hashed(C.c_int64(0), C.c_int64(n), C.c_int64(bins), C.c_int64(5), want.ctypes.data_as(C.POINTER(C.c_int64)))
    for _, _, h in res:
        assert np.array_equal(h, want)


def _heat_box_rank(rank, world, port, rows, cols, iters, q):
    """each rank uploads and downloads only its own chunk's box (mt_array_*_box_async)"""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    ctx = mb.context(workers=world, devices=1, worker_rank=rank, gpu_base=0)
    ctx.connect_peers()
    devs = ctx.devices
    dist_ = lambda: ctx.dist.stencil([rows, cols], [rows // world, cols], [1, 0], devs)  # noqa: E731
    a = ctx.create_array([rows, cols], "f32", dist_(), 0)
    b = ctx.create_array([rows, cols], "f32", dist_(), 0)
    work = ctx.dist.block_work([rows, cols], [16, 16], [rows // world, cols], devs)
    mine = [c for c in ctx.chunks(a) if c.home[0] == rank][0]
    box = (mine.lo, mine.hi)
    full = np.random.default_rng(11).standard_normal((rows, cols)).astype(np.float32)
    host_in = torch.from_numpy(full[mine.lo[0]:mine.hi[0]].copy()).pin_memory()
    host_out = torch.full((mine.hi[0] - mine.lo[0], cols), float("nan"), dtype=torch.float32).pin_memory()
    ctx.write_async(a, host_in, box=box)
    for _ in range(iters):
        ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
        a, b = b, a
    ctx.read_async(a, host_out, box=box)
    ctx.synchronize()
    per = rows // world
    lo = 0 if rank == 0 else rank * per + 1  # rows this rank's read tasks cover (lowest-id chunk)
    hi = min(rows, (rank + 1) * per + 1)
    q.put((rank, host_out.numpy()[lo - mine.lo[0]:hi - mine.lo[0]].copy(), lo, hi))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def test_two_process_box_host_io_matches_single_process():
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    rows, cols, iters, world = 256, 512, 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_heat_box_rank, args=(r, world, port, rows, cols, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert [(p[2], p[3]) for p in parts] == [(0, rows // 2 + 1), (rows // 2 + 1, rows)]
    got = np.concatenate([p[1] for p in parts])
    full = np.random.default_rng(11).standard_normal((rows, cols)).astype(np.float32)
    with mb.context(workers=1, devices=world, num_gpus=1) as c:
        devs = c.devices
        a = c.create_array([rows, cols], "f32", c.dist.stencil([rows, cols], [rows // world, cols], [1, 0], devs), 0)
        b = c.create_array([rows, cols], "f32", c.dist.stencil([rows, cols], [rows // world, cols], [1, 0], devs), 0)
        w = c.dist.block_work([rows, cols], [16, 16], [rows // world, cols], devs)
        c.write(a, full)
        for _ in range(iters):
            c.launch("heat2d", [rows, cols], [16, 16], w, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
            a, b = b, a
        want = c.read(a)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def _silent_peer_rank(rank, world, port, q):
    """rank 1 never launches, so rank 0's halo receive has no sender: the bounded GPU-side wait
    must turn that into an execution error instead of a hung GPU"""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), MTB_PEER_TIMEOUT_S="2")
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    rows, cols = 64, 128
    ctx = mb.context(workers=world, devices=1, worker_rank=rank, gpu_base=0)
    ctx.connect_peers()
    outcome = "ok"
    if rank == 0:
        devs = ctx.devices
        dist_ = lambda: ctx.dist.stencil([rows, cols], [rows // world, cols], [1, 0], devs)  # noqa: E731
        a = ctx.create_array([rows, cols], "f32", dist_(), 0)
        b = ctx.create_array([rows, cols], "f32", dist_(), 0)
        work = ctx.dist.block_work([rows, cols], [16, 16], [rows // world, cols], devs)
        ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
        try:
            ctx.synchronize()
            outcome = "returned"
        except mb.MantaError as e:
            outcome = type(e).__name__
    q.put((rank, outcome))
    dist.barrier()
    if rank != 0:
        ctx.close()
    dist.destroy_process_group()
    os._exit(0)  # rank 0's CUDA context is poisoned by the trap: skip teardown


def test_missing_peer_message_times_out():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_silent_peer_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    assert res[0] == "ExecutionError"


def test_four_process_heat_matches_single_process():
    """four ranks: the interior ones exchange halo rows with two neighbours each; enough steps
    to wrap every peer ring several times"""
    stats = _two_process_heat(512, 1024, 40, world=4)
    assert all(s["bytes_sent"] > 0 and s["bytes_received"] > 0 for s in stats)
