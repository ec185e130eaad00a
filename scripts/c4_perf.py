#!/usr/bin/env python
"""BASELINE config C4 on one B200 through the framework: histogram (n i32 values, reduce(+)
into i64 bins) and int32 k-means (assign + update + finalize). Device-event timings, one JSON
line per workload."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(ctx, kernel, fn, steps):
    fn()
    ctx.synchronize()
    ctx.profile_kernels(True)
    k0, m0 = ctx.kernel_time(kernel)
    ctx.mark(0)
    for _ in range(steps):
        fn()
    ctx.mark(1)
    ms = ctx.elapsed_ms()
    ctx.synchronize()
    ctx.profile_kernels(False)
    k1, m1 = ctx.kernel_time(kernel)
    return ms / steps, (m1 - m0) / max(1, k1 - k0)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--hist-n", type=int, default=4_000_000_000)
    p.add_argument("--km-n", type=int, default=1_000_000_000)
    p.add_argument("--steps", type=int, default=5)
    args = p.parse_args()
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        hbm = json.load(f)["hbm_gbs"]
    ctx = mb.context(workers=1, devices=1, num_gpus=1)
    dev = ctx.devices
    n = args.hist_n
    for bins in (256, 65536):
        x = ctx.create_array([n], "i32", ctx.dist.single([n], dev[0]), 0)
        h = ctx.create_array([bins], "i64", ctx.dist.single([bins], dev[0]), 0)
        w = ctx.dist.block_work([n], [256], [n], dev)
        ctx.launch("hpattern1d", [n], [256], w, [n, bins, 12345, Arr(x)], "global i => write out[i]")

        def step():
            ctx.launch("histogram", [n], [256], w, [n, bins, Arr(x), Arr(h)], "global i => read x[i], reduce(+) hist[:]")
            ctx.flush()

        ms, kms = timed(ctx, "histogram", step, args.steps)
        total = int(ctx.read(h).sum())
        print(json.dumps({"workload": f"histogram n={n} bins={bins}", "ms_per_step": ms, "kernel_ms": kms, "elements_per_s": n / (ms / 1e3),
                          "achieved_gbs": 4 * n / (kms / 1e3) / 1e9, "frac_of_hbm": 4 * n / (kms / 1e3) / 1e9 / hbm, "count_check": total == n}), flush=True)
        ctx.delete_array(x)
        ctx.delete_array(h)
        ctx.synchronize()

    if args.km_n <= 0:
        return
    n, k, d = args.km_n, 256, 16
    pts = ctx.create_array([n, d], "i32", ctx.dist.single([n, d], dev[0]), 0)
    asg = ctx.create_array([n], "i32", ctx.dist.single([n], dev[0]), 0)
    cen = ctx.create_array([k, d], "i32", ctx.dist.single([k, d], dev[0]), 0)
    sums = ctx.create_array([k, d], "i64", ctx.dist.single([k, d], dev[0]), 0)
    cnts = ctx.create_array([k], "i64", ctx.dist.single([k], dev[0]), 0)
    ctx.launch("ipattern2d_i32", [n, d], [256, 16], ctx.dist.block_work([n, d], [256, 16], [n, d], dev), [n, d, 1000, Arr(pts)],
               "global [i, j] => write out[i,j]")
    wk = ctx.dist.block_work([k, d], [16, 16], [k, d], dev)
    ctx.launch("ipattern2d_i32", [k, d], [16, 16], wk, [k, d, 997, Arr(cen)], "global [i, j] => write out[i,j]")
    w1 = ctx.dist.block_work([n], [256], [n], dev)

    def assign():
        ctx.launch("kmeans_assign_i32", [n], [256], w1, [n, k, d, Arr(asg), Arr(pts), Arr(cen)],
                   "global i => write assign[i], read points[i,:], read centroids[:,:]")
        ctx.flush()

    def update():
        ctx.launch("kmeans_update_i32", [n], [256], w1, [n, d, Arr(pts), Arr(asg), Arr(sums), Arr(cnts)],
                   "global i => read points[i,:], read assign[i], reduce(+) sums[:,:], reduce(+) counts[:]")
        ctx.flush()

    ms, kms = timed(ctx, "kmeans_assign_i32", assign, 2)
    ops = 3.0 * n * k * d
    print(json.dumps({"workload": f"kmeans_assign_i32 n={n} k={k} d={d}", "ms_per_step": ms, "kernel_ms": kms, "int_ops_per_s": ops / (kms / 1e3)}), flush=True)
    ms, kms = timed(ctx, "kmeans_update_i32", update, args.steps)
    byts = n * (d + 1) * 4
    print(json.dumps({"workload": f"kmeans_update_i32 n={n} d={d}", "ms_per_step": ms, "kernel_ms": kms, "achieved_gbs": byts / (kms / 1e3) / 1e9,
                      "frac_of_hbm": byts / (kms / 1e3) / 1e9 / hbm, "count_check": int(ctx.read(cnts).sum()) == n}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
