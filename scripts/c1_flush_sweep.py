#!/usr/bin/env python
"""C1 (heat2d 4096^2, 4 chunks, 100 iterations): device time per iteration as a function of how
many launches are handed to the executor per flush (1 = the bench's one flush per launch)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2202_05549_b200 as mb  # noqa: E402
from paper_2202_05549_b200 import Arr  # noqa: E402

rows = cols = 4096
iters = 100
for per in [int(x) for x in (sys.argv[1:] or ["1", "2", "4", "10", "100"])]:
    with mb.context(workers=1, devices=4, num_gpus=1, retain_plan=False) as ctx:
        a, b, work = bench.setup_heat(ctx, rows, cols, 4)

        def run(n):
            global a, b
            for i in range(n):
                ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, bench.ALPHA, Arr(b), Arr(a)], bench.ANN)
                if (i + 1) % per == 0:
                    ctx.flush()
                a, b = b, a
            ctx.flush()

        for _ in range(3):
            run(iters)
        ctx.synchronize()
        best = 1e9
        for _ in range(5):
            ctx.mark(0)
            t0 = time.perf_counter()
            run(iters)
            host = time.perf_counter() - t0
            ctx.mark(1)
            best = min(best, ctx.elapsed_ms() / iters)
            ctx.synchronize()
        st = ctx.exec_stats()
        print(json.dumps({"launches_per_flush": per, "ms_per_iter": best, "host_ms_per_iter": host * 1e3 / iters,
                          "frac_hbm": 8 * rows * cols / 6553e9 * 1e3 / best, "captures": st.get("graph_captures"), "replays": st.get("graph_replays")}))
