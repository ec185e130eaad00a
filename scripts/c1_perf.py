#!/usr/bin/env python
"""BASELINE config C1 (the reference's CPU-runnable case) on one B200: heat2d 4096^2 f32,
100 iterations, stencil distribution into 4 chunks (4 logical devices on the GPU), one
distributed launch per iteration. Device-event time and host time per iteration."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2202_05549_b200 as mb  # noqa: E402
from paper_2202_05549_b200 import Arr  # noqa: E402

rows = cols = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 4
iters = 100
with mb.context(workers=1, devices=chunks, num_gpus=1, retain_plan=False) as ctx:
    a, b, work = bench.setup_heat(ctx, rows, cols, chunks)
    ctx.synchronize()

    def run(n):
        global a, b
        for _ in range(n):
            ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, bench.ALPHA, Arr(b), Arr(a)], bench.ANN)
            ctx.flush()
            a, b = b, a

    run(20)
    ctx.synchronize()
    ctx.mark(0)
    t0 = time.perf_counter()
    run(iters)
    host = time.perf_counter() - t0
    ctx.mark(1)
    ms = ctx.elapsed_ms()
    ctx.synchronize()
    ideal = 8 * rows * cols / 6553e9 * 1e3
    print(json.dumps({"workload": f"heat2d {rows}^2 x{iters}, {chunks} chunks", "ms_per_iter": ms / iters, "host_ms_per_iter": host * 1e3 / iters,
                      "cell_updates_per_s": rows * cols * iters / (ms / 1e3), "hbm_bound_ms_per_iter": ideal}))
