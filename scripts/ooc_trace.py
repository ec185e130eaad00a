#!/usr/bin/env python
"""Small out-of-core heat2d run with the spill tier's decisions traced (MTB_SPILL_TRACE): 16
chunks of 16 MiB per array, device capped at 10 chunks, per-iteration traffic vs the minimum."""
import os
import sys

os.environ["MTB_SPILL_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

cols, cr, nch = 16384, 256, 16
r = bench.run_ooc(nch * cr, cols, cr, 10 * cr * cols * 4 / 2**30, 1.0, 6, 2)
print({k: r[k] for k in ("h2d_gib_per_iter", "d2h_gib_per_iter", "min_gib_each_way_per_iter", "time_over_bound", "evictions")})
