#!/usr/bin/env python
"""Out-of-core heat2d (BASELINE config C5 analog) on one B200 with the pinned-host spill tier;
the measurement itself is bench.run_ooc (also the bench's `out_of_core` leg). Prints one JSON
line."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


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
    import bench
    print(json.dumps(bench.run_ooc(args.rows, args.cols, args.chunk_rows, args.capacity_gib, args.host_gib, args.iters, args.warmup, args.lookahead)))


if __name__ == "__main__":
    main()
