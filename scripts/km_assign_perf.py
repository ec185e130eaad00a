"""k-means assign (BASELINE C4: int32 points, d=16, k=256) kernel time through the framework for
the variants selected by MTB_KM_VARIANT (set by the caller), with a sha256 of the assignments so
variants can be compared for bit-identity. Usage: MTB_KM_VARIANT=v python scripts/km_assign_perf.py [n]"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000_000
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    k, d = 256, 16
    with mb.context(workers=1, devices=1, num_gpus=1) as ctx:
        dev = ctx.devices
        pts = ctx.create_array([n, d], "i32", ctx.dist.single([n, d], dev[0]), 0)
        asg = ctx.create_array([n], "i32", ctx.dist.single([n], dev[0]), 0)
        cen = ctx.create_array([k, d], "i32", ctx.dist.single([k, d], dev[0]), 0)
        ctx.launch("ipattern2d_i32", [n, d], [256, 16], ctx.dist.block_work([n, d], [256, 16], [n, d], dev), [n, d, 1000, Arr(pts)],
                   "global [i, j] => write out[i,j]")
        ctx.launch("ipattern2d_i32", [k, d], [16, 16], ctx.dist.block_work([k, d], [16, 16], [k, d], dev), [k, d, 997, Arr(cen)],
                   "global [i, j] => write out[i,j]")
        w1 = ctx.dist.block_work([n], [256], [n], dev)

        def assign():
            ctx.launch("kmeans_assign_i32", [n], [256], w1, [n, k, d, Arr(asg), Arr(pts), Arr(cen)],
                       "global i => write assign[i], read points[i,:], read centroids[:,:]")
            ctx.flush()

        assign()
        ctx.synchronize()
        ctx.profile_kernels(True)
        for _ in range(3):
            assign()
        ctx.synchronize()
        cnt, ms = ctx.kernel_time("kmeans_assign_i32")
        a = ctx.read(asg)
    kms = ms / cnt
    terms = float(n) * k * d
    print(json.dumps({"variant": os.environ.get("MTB_KM_VARIANT", "0"), "n": n, "kernel_ms": kms, "ms_per_1e9": kms * 1e9 / n,
                      "frac_nominal_ffma": terms / (kms / 1e3) / (148 * 128 * 1.965e9), "sha256": hashlib.sha256(a.tobytes()).hexdigest()[:16]}))


if __name__ == "__main__":
    main()
