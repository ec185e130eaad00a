#!/usr/bin/env python
"""Out-of-core heat2d (BASELINE config C5 analog) on one B200 with the pinned-host spill tier.

Working set = 2 arrays of rows x 65536 f32 in 1 GiB chunks (4096 rows, halo [1,0]); the
device capacity is capped at `--capacity-gib`. Per iteration the minimum traffic is about
(working set - capacity) each way; the bound is that volume over the measured pinned
H2D/D2H bandwidth (both directions concurrently, full duplex). Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def link_bandwidth(gib=4):
    import torch
    n = gib << 30
    h_src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_src = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, fn in [("h2d", lambda: d_dst.copy_(h_src, non_blocking=True)), ("d2h", lambda: h_dst.copy_(d_src, non_blocking=True))]:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        res[name] = 3 * n / (time.perf_counter() - t0) / 1e9
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        with torch.cuda.stream(s1):
            d_dst.copy_(h_src, non_blocking=True)
        with torch.cuda.stream(s2):
            h_dst.copy_(d_src, non_blocking=True)
    torch.cuda.synchronize()
    res["duplex_each_way"] = 3 * n / (time.perf_counter() - t0) / 1e9
    del h_src, h_dst, d_src, d_dst
    torch.cuda.empty_cache()
    return res


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=int, default=98304)  # 2 x 24 GiB
    p.add_argument("--cols", type=int, default=65536)
    p.add_argument("--chunk-rows", type=int, default=4096)
    p.add_argument("--capacity-gib", type=float, default=32.0)
    p.add_argument("--host-gib", type=float, default=64.0)
    p.add_argument("--iters", type=int, default=4)
    p.add_argument("--warmup", type=int, default=2)
    p.add_argument("--lookahead", type=int, default=0)
    args = p.parse_args()
    bw = link_bandwidth()
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    rows, cols, cr = args.rows, args.cols, args.chunk_rows
    cap = int(args.capacity_gib * (1 << 30))
    la = args.lookahead or 3 * (rows // cr) * 3
    ctx = mb.context(workers=1, devices=1, num_gpus=1, device_capacity=cap, host_capacity=int(args.host_gib * (1 << 30)), lookahead_tasks=la)
    devs = ctx.devices
    dist = lambda: ctx.dist.stencil([rows, cols], [cr, cols], [1, 0], devs)  # noqa: E731
    a = ctx.create_array([rows, cols], "f32", dist(), 0)
    b = ctx.create_array([rows, cols], "f32", dist(), 0)
    work = ctx.dist.block_work([rows, cols], [16, 16], [cr, cols], devs)
    ctx.launch("ramp2d_f32", [rows, cols], [16, 16], work, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
    ann = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"
    t_setup = time.perf_counter()
    for _ in range(args.warmup):
        ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], ann)
        ctx.flush()
        a, b = b, a
    ctx.synchronize()
    t_setup = time.perf_counter() - t_setup
    s0 = ctx.exec_stats()
    ctx.mark(0)
    for _ in range(args.iters):
        ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, 0.1, Arr(b), Arr(a)], ann)
        ctx.flush()
        a, b = b, a
    ctx.mark(1)
    ms = ctx.elapsed_ms()
    ctx.synchronize()
    s1 = ctx.exec_stats()
    ws = 2 * rows * cols * 4
    h2d = (s1["spill_bytes_h2d"] - s0["spill_bytes_h2d"]) / args.iters
    d2h = (s1["spill_bytes_d2h"] - s0["spill_bytes_d2h"]) / args.iters
    # each iteration reads one array and overwrites the other; the overwritten one is dead, so
    # at steady state only the part of an array that does not fit must cross the link each way
    minimum = max(0, ws // 2 - cap)
    survey_bound = max(0, ws - cap)  # SURVEY 8d's (working set - resident) each way
    per_iter = ms / args.iters / 1e3
    bound = minimum / (bw["duplex_each_way"] * 1e9)
    out = {"workload": f"out-of-core heat2d {rows}x{cols} f32 x2 arrays, {cr}-row chunks, device capacity {args.capacity_gib} GiB",
           "working_set_gib": ws / 2**30, "capacity_gib": args.capacity_gib, "iters": args.iters, "s_per_iter": per_iter,
           "cell_updates_per_s": rows * cols / per_iter, "h2d_gib_per_iter": h2d / 2**30, "d2h_gib_per_iter": d2h / 2**30,
           "min_gib_each_way_per_iter": minimum / 2**30, "moved_over_min": max(h2d, d2h) / minimum if minimum else None,
           "survey_bound_gib_each_way": survey_bound / 2**30,
           "time_over_survey_bound": per_iter / (survey_bound / (bw["duplex_each_way"] * 1e9)) if survey_bound else None,
           "link_gbs": bw, "bound_s_per_iter": bound, "time_over_bound": per_iter / bound if bound else None,
           "lookahead_tasks": la, "warmup_s": t_setup, "evictions": s1["evictions"] - s0["evictions"]}
    print(json.dumps(out))
    ctx.close()


if __name__ == "__main__":
    main()
