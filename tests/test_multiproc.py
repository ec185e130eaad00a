"""Host-side logic of the one-process-per-GPU mode, on CPU with gloo (world_size 2).

Every rank runs the same deterministic planner (no driver->worker RPC, unlike the paper's
MPI driver): the plans must be byte-identical across ranks, and the
per-worker task subsets must partition the plan with every dependency local to its worker
and every send matched by exactly one recv on the peer (tags per (src, dst) pair).
"""
import hashlib
import json
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _plan_on_rank(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    ctx = mb.context(workers=world, devices=1, execute=False)
    n = 1 << 12
    devs = ctx.devices
    a = ctx.create_array([n, 64], "f32", ctx.dist.stencil([n, 64], [n // world, 64], [1, 0], devs), 1)
    b = ctx.create_array([n, 64], "f32", ctx.dist.stencil([n, 64], [n // world, 64], [1, 0], devs), 0)
    w = ctx.dist.block_work([n, 64], [16, 16], [n // world, 64], devs)
    for _ in range(3):
        ctx.launch("heat2d", [n, 64], [16, 16], w, [n, 64, 0.1, Arr(b), Arr(a)], "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]")
        a, b = b, a
    plan = ctx.plan()
    digest = hashlib.sha256(json.dumps(plan).encode()).hexdigest()
    digests = [None] * world
    dist.all_gather_object(digests, digest)
    mine = [t for t in plan if t["worker"] == rank]
    counts = [None] * world
    dist.all_gather_object(counts, len(mine))
    q.put((rank, digests, counts, plan if rank == 0 else None))
    dist.destroy_process_group()


def test_replicated_planning_is_identical_across_ranks():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_plan_on_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    digests = results[0][1]
    assert len(set(digests)) == 1
    plan = results[0][3]
    assert sum(results[0][2]) == len(plan)
    worker_of = {t["id"]: t["worker"] for t in plan}
    for t in plan:
        assert all(worker_of[d] == t["worker"] for d in t["deps"])
    sends = {(t["worker"], t["peer"], t["tag"]) for t in plan if t["kind"] == "send"}
    recvs = {(t["peer"], t["worker"], t["tag"]) for t in plan if t["kind"] == "recv"}
    assert sends == recvs and len(sends) == 2 * 3  # 2(P-1) halo messages per iteration


def _collective_plan_on_rank(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    ctx = mb.context(workers=world, devices=2, execute=False, collective_reduce=True)
    devs = ctx.devices
    n, k, d = 4096, 8, 4
    pts = ctx.create_array([n, d], "i32", ctx.dist.row([n, d], n // len(devs), devs), 1)
    asg = ctx.create_array([n], "i32", ctx.dist.row([n], n // len(devs), devs), 0)
    sums = ctx.create_array([k, d], "i64", ctx.dist.replicated([k, d], devs), 0)
    cnts = ctx.create_array([k], "i64", ctx.dist.replicated([k], devs), 0)
    w = ctx.dist.block_work([n], [64], [n // len(devs)], devs)
    for _ in range(2):
        ctx.launch("kmeans_update_i32", [n], [64], w, [n, d, Arr(pts), Arr(asg), Arr(sums), Arr(cnts)],
                   "global i => read points[i,:], read assign[i], reduce(+) sums[:,:], reduce(+) counts[:]")
    plan = ctx.plan()
    digest = hashlib.sha256(json.dumps(plan).encode()).hexdigest()
    digests = [None] * world
    dist.all_gather_object(digests, digest)
    mine = [t["tag"] for t in plan if t["worker"] == rank and t["kind"] == "allreduce"]
    seqs = [None] * world
    dist.all_gather_object(seqs, mine)
    q.put((rank, digests, seqs))
    dist.destroy_process_group()


def test_collective_groups_line_up_across_ranks():
    """NCCL needs every rank to enter the same collectives in the same order: each worker's
    allreduce tasks, in its own issue order, must walk the same group sequence"""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_collective_plan_on_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    digests, seqs = results[0][1], results[0][2]
    assert len(set(digests)) == 1
    assert seqs[0] == seqs[1] == [0, 1, 2, 3]  # 2 launches x (sums, counts)
