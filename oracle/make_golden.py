#!/usr/bin/env python
"""ORACLE / TEST INFRASTRUCTURE: generates tests/golden/ from the reference itself.

Run here (where /root/reference exists) after `make -C oracle`:
    python oracle/make_golden.py

Writes
  scenarios.json        the reference's bundled scenarios (proj/scenarios/*.json), verbatim data
  scenario_outputs.json per scenario: the reference run_scenario oracle-mode result of every
                        array (sha256 of the bytes, shape, dtype, and the values when small)
  plans.json            the reference driver's plan (tasks incl. deps) for every bundled
                        scenario on its own system shape and in oracle mode
  kernels.npz           small known-answer vectors from the reference CPU executor for the
                        kernels restated through its plugin API (heat2d, histogram, int32 k-means)
Every value comes from oracle/_ref/libmanta_ref.so (the unmodified reference + ref_shim.cpp).
"""
from __future__ import annotations

import glob
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden")
SCEN_DIR = "/root/reference/proj/scenarios"


def main():
    import oracle
    from paper_2202_05549_b200 import Arr
    from paper_2202_05549_b200 import scenario as S
    from oracle import scenario as R
    ref = oracle.reference()
    os.makedirs(OUT, exist_ok=True)

    scen = {}
    for f in sorted(glob.glob(os.path.join(SCEN_DIR, "*.json"))):
        with open(f) as fh:
            scen[os.path.basename(f)[:-5]] = json.load(fh)
    with open(os.path.join(OUT, "scenarios.json"), "w") as fh:
        json.dump(scen, fh, indent=1, sort_keys=True)

    outputs, plans = {}, {}
    for name, sc in scen.items():
        res, coherent = R.run(ref, sc, oracle_mode=True)
        outputs[name] = {"coherent": coherent, "arrays": {}}
        for an, arr in res.items():
            e = {"shape": list(arr.shape), "dtype": str(arr.dtype), "sha256": hashlib.sha256(arr.tobytes()).hexdigest()}
            if arr.size <= 4096:
                e["values"] = arr.ravel().tolist()
            outputs[name]["arrays"][an] = e
        plans[name] = {"system": R.plan(ref, sc).dicts(), "oracle": R.plan(ref, sc, oracle_mode=True).dicts()}
    with open(os.path.join(OUT, "scenario_outputs.json"), "w") as fh:
        json.dump(outputs, fh, indent=1, sort_keys=True)
    with open(os.path.join(OUT, "plans.json"), "w") as fh:
        json.dump(plans, fh, separators=(",", ":"), default=list)

    # known-answer vectors for the restated kernels, from the reference executor (2x2 system)
    vec = {}
    rows, cols, iters = 40, 24, 3
    ctx = oracle.reference_context(workers=2, devices=2, execute=True)
    devs = ctx.devices
    dist = lambda: ctx.dist.stencil([rows, cols], [10, cols], [1, 0], devs)  # noqa: E731
    a = ctx.create_array([rows, cols], "f32", dist(), 0)
    b = ctx.create_array([rows, cols], "f32", dist(), 0)
    work = ctx.dist.block_work([rows, cols], [5, 8], [10, cols], devs)
    ctx.launch("ramp2d_f32", [rows, cols], [5, 8], work, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
    vec["heat_in"] = ctx.read(a)
    for _ in range(iters):
        ctx.launch("heat2d", [rows, cols], [5, 8], work, [rows, cols, 0.1, Arr(b), Arr(a)], "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]")
        a, b = b, a
    ctx.synchronize()
    vec["heat_out"] = ctx.read(a)
    ctx.close()

    n, bins = 5000, 64
    ctx = oracle.reference_context(workers=2, devices=2, execute=True)
    devs = ctx.devices
    x = ctx.create_array([n], "i32", ctx.dist.row([n], 1250, devs), 0)
    h = ctx.create_array([bins], "i64", ctx.dist.replicated([bins], devs), 0)
    ctx.launch("hpattern1d", [n], [64], ctx.dist.block_work([n], [64], [1280], devs), [n, bins, 12345, Arr(x)], "global i => write out[i]")
    ctx.launch("histogram", [n], [64], ctx.dist.block_work([n], [64], [1280], devs), [n, bins, Arr(x), Arr(h)],
               "global i => read x[i], reduce(+) hist[:]")
    ctx.synchronize()
    vec["hist_x"], vec["hist_out"] = ctx.read(x), ctx.read(h)
    ctx.close()

    n, k, d = 600, 8, 16
    ctx = oracle.reference_context(workers=2, devices=2, execute=True)
    devs = ctx.devices
    pts = ctx.create_array([n, d], "i32", ctx.dist.row([n, d], 150, devs), 0)
    asg = ctx.create_array([n], "i32", ctx.dist.row([n], 150, devs), 0)
    cen = ctx.create_array([k, d], "i32", ctx.dist.replicated([k, d], devs), 0)
    sums = ctx.create_array([k, d], "i64", ctx.dist.replicated([k, d], devs), 0)
    cnts = ctx.create_array([k], "i64", ctx.dist.replicated([k], devs), 0)
    wp = ctx.dist.block_work([n, d], [16, 16], [160, d], devs)
    ctx.launch("ipattern2d_i32", [n, d], [16, 16], wp, [n, d, 1000, Arr(pts)], "global [i, j] => write out[i,j]")
    ctx.launch("ipattern2d_i32", [k, d], [8, 16], ctx.dist.block_work([k, d], [8, 16], [8, d], devs), [k, d, 997, Arr(cen)],
               "global [i, j] => write out[i,j]")
    w1 = ctx.dist.block_work([n], [64], [192], devs)
    for _ in range(3):
        ctx.launch("kmeans_assign_i32", [n], [64], w1, [n, k, d, Arr(asg), Arr(pts), Arr(cen)],
                   "global i => write assign[i], read points[i,:], read centroids[:,:]")
        ctx.launch("kmeans_update_i32", [n], [64], w1, [n, d, Arr(pts), Arr(asg), Arr(sums), Arr(cnts)],
                   "global i => read points[i,:], read assign[i], reduce(+) sums[:,:], reduce(+) counts[:]")
        ctx.launch("kmeans_finalize_i32", [k, d], [8, 16], ctx.dist.block_work([k, d], [8, 16], [8, d], devs), [k, d, Arr(cen), Arr(sums), Arr(cnts)],
                   "global [i, j] => readwrite centroids[i,j], read sums[i,j], read counts[i]")
    ctx.synchronize()
    vec["km_points"], vec["km_assign"], vec["km_centroids"] = ctx.read(pts), ctx.read(asg), ctx.read(cen)
    vec["km_sums"], vec["km_counts"] = ctx.read(sums), ctx.read(cnts)
    ctx.close()
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **vec)
    print("golden written to", OUT)


if __name__ == "__main__":
    main()
