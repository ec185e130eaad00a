"""nbody_like (f64 all-pairs) throughput on one B200 through the planner: pair interactions/s."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2202_05549_b200 as mb  # noqa: E402
from paper_2202_05549_b200 import Arr  # noqa: E402

n, d = int(sys.argv[1]) if len(sys.argv) > 1 else 65536, 3
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
with mb.context(workers=1, devices=1, num_gpus=1) as ctx:
    dv = ctx.devices
    p = ctx.create_array([n, d], "f64", ctx.dist.single([n, d], dv[0]), 0)
    f = ctx.create_array([n, d], "f64", ctx.dist.single([n, d], dv[0]), 0)
    ctx.write(p, np.random.default_rng(1).standard_normal((n, d)))
    w = ctx.dist.block_work([n], [256], [n], dv)

    def step():
        ctx.launch("nbody_like", [n], [256], w, [n, d, Arr(f), Arr(p)], "global i => write force[i,:], read pos[:,:]")
        ctx.flush()

    step()
    ctx.synchronize()
    ctx.mark(0)
    for _ in range(steps):
        step()
    ctx.mark(1)
    ms = ctx.elapsed_ms() / steps
    print(f"nbody n={n} d={d}: {ms:.2f} ms/step, {n * (n - 1) / (ms / 1e3) / 1e9:.1f} G pair-interactions/s")
