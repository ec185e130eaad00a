"""Plan-only cost of band-reads of one chunk: S superblocks read/write
bands of single-chunk 65536^2 arrays (heat2d) or one single-chunk 1D x (histogram).
Prints ms per launch for region and compat dependency modes. No GPU needed."""
import sys
import time

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr


def heat(S, compat, launches=4):
    n = 65536
    with mb.context(workers=1, devices=1, execute=False, compat_deps=compat, plan_cache=False) as ctx:
        devs = ctx.devices
        dist = lambda: ctx.dist.single([n, n], devs[0])  # noqa: E731
        a = ctx.create_array([n, n], "f32", dist(), 0)
        b = ctx.create_array([n, n], "f32", dist(), 0)
        work = ctx.dist.block_work([n, n], [16, 16], [n // S, n], devs)
        ann = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"
        ts = []
        for _ in range(launches):
            t0 = time.perf_counter()
            ctx.launch("heat2d", [n, n], [16, 16], work, [n, n, 0.1, Arr(b), Arr(a)], ann)
            ts.append(time.perf_counter() - t0)
            a, b = b, a
        return min(ts[1:]) * 1e3


def hist(S, compat, launches=4):
    n = 1 << 32
    bins = 256
    with mb.context(workers=1, devices=1, execute=False, compat_deps=compat, plan_cache=False) as ctx:
        devs = ctx.devices
        x = ctx.create_array([n], "i32", ctx.dist.single([n], devs[0]), 0)
        h = ctx.create_array([bins], "i64", ctx.dist.single([bins], devs[0]), 0)
        work = ctx.dist.block_work([n], [256], [n // S], devs)
        ann = "global [i] => read x[i], reduce(+) hist[:]"
        ts = []
        for _ in range(launches):
            t0 = time.perf_counter()
            ctx.launch("histogram", [n], [256], work, [n, bins, Arr(x), Arr(h)], ann)
            ts.append(time.perf_counter() - t0)
        return min(ts[1:]) * 1e3


if __name__ == "__main__":
    sizes = [int(s) for s in sys.argv[1:]] or [256, 512, 1024]
    for S in sizes:
        print(f"S={S:5d} heat region {heat(S, False):8.2f} ms  compat {heat(S, True):8.2f} ms | "
              f"hist region {hist(S, False):8.2f} ms  compat {hist(S, True):8.2f} ms", flush=True)
