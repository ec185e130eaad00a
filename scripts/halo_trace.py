"""Two-process (one worker per process) heat2d with 3 superblocks per rank (top strip, interior,
bottom strip), per-task device timestamps on (mt_exec_trace): shows the interior superblock
overlapping the halo send/recv of the same iteration, and the duration of each message task.

    python scripts/halo_trace.py [rows] [cols] [iters] [out_dir]
    python scripts/halo_trace.py latency [cols] [iters] [out_dir]

The latency form runs a 64-row grid (32 rows per rank: a few-microsecond kernel) so an
iteration is dominated by the halo exchange (one row each way, cols x 4 bytes), and reports the
time per iteration over `iters` iterations (device-synchronized wall clock, max over ranks).

Writes <out_dir>/halo_trace_rank<r>.json (the executor's run_report with task records) and
prints a per-iteration overlap summary. With both ranks on ONE GPU (no MPS) the two processes'
kernels time-slice, so cross-process latency includes context switches; the within-rank overlap
of the interior with the message kernels is what this demonstrates."""
import json
import os
import socket
import sys

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
HEAT = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"


def latency_main(rank, world, port, cols, iters, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import time

    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    rows = 64
    ctx = mb.context(workers=world, devices=1, worker_rank=rank, gpu_base=rank % torch.cuda.device_count(), retain_plan=False)
    ctx.connect_peers()
    a, b, work = bench.setup_heat(ctx, rows, cols, world)

    def run(n):
        nonlocal a, b
        for _ in range(n):
            ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
            ctx.flush()
            a, b = b, a
        ctx.synchronize()

    run(20)
    dist.barrier()
    t0 = time.perf_counter()
    run(iters)
    dt = bench.barrier_max(time.perf_counter() - t0, world)
    st = ctx.exec_stats()
    if rank == 0:
        res = {"mode": "latency", "rows": rows, "cols": cols, "halo_bytes_each_way": cols * 4, "iters": iters, "us_per_iteration": dt / iters * 1e6,
               "message_ops_per_message": st["message_ops"] / max(1, st["messages"])}
        print(json.dumps(res), flush=True)
        with open(os.path.join(out_dir, "halo_latency.json"), "w") as fh:
            json.dump(res, fh)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def rank_main(rank, world, port, rows, cols, iters, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    gpu = rank % torch.cuda.device_count()
    ctx = mb.context(workers=world, devices=1, worker_rank=rank, gpu_base=gpu)
    ctx.connect_peers()
    a, b, work = bench.setup_heat(ctx, rows, cols, world, strip=128)
    for _ in range(3):  # warm-up
        ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
        a, b = b, a
    ctx.synchronize()
    dist.barrier()
    ctx.trace(True)
    first = None
    for i in range(iters):
        f, _ = ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
        first = f if first is None else first
        ctx.flush()
        a, b = b, a
    ctx.synchronize()
    rep = json.loads(ctx.report_json())
    st = ctx.exec_stats()
    with open(os.path.join(out_dir, f"halo_trace_rank{rank}.json"), "w") as fh:
        json.dump({"rank": rank, "report": rep, "stats": st}, fh)
    recs = [r for w in rep["workers"] for r in w["tasks"]]
    execs = [r for r in recs if r["kind"] == "execute"]
    msgs = [r for r in recs if r["kind"] in ("send", "recv")]
    lines = []
    # per iteration: executes come in (top, interior, bottom) order per rank
    for it in range(iters):
        ex = execs[3 * it:3 * it + 3]
        if len(ex) < 3:
            break
        interior = ex[1]
        mine = [m for m in msgs if m["id"] > ex[0]["id"] - 8 and m["id"] < ex[2]["id"] + 8]
        ov = [m for m in mine if m["start_ns"] < interior["end_ns"] and m["end_ns"] > interior["start_ns"]]
        lines.append({"iteration": it, "interior_us": (interior["end_ns"] - interior["start_ns"]) / 1e3,
                      "messages": [(m["kind"], round((m["end_ns"] - m["start_ns"]) / 1e3, 1)) for m in mine],
                      "overlapping_interior": len(ov)})
    print(json.dumps({"rank": rank, "message_ops_per_message": st["message_ops"] / max(1, st["messages"]), "iterations": lines}), flush=True)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    latency = len(sys.argv) > 1 and sys.argv[1] == "latency"
    argv = sys.argv[1:] if latency else sys.argv
    rows = 64 if latency else (int(argv[1]) if len(argv) > 1 else 8192)
    cols = int(argv[2 - latency]) if len(argv) > 2 - latency else 65536
    iters = int(argv[3 - latency]) if len(argv) > 3 - latency else (500 if latency else 6)
    out_dir = argv[4 - latency] if len(argv) > 4 - latency else os.path.join(ROOT, "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    ctx = mp.get_context("spawn")
    if latency:
        procs = [ctx.Process(target=latency_main, args=(r, world, port, cols, iters, out_dir)) for r in range(world)]
    else:
        procs = [ctx.Process(target=rank_main, args=(r, world, port, rows, cols, iters, out_dir)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        if p.exitcode != 0:
            sys.exit(1)
