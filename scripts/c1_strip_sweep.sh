#!/bin/bash
# C1 (4096^2, 4 chunks) with halo-facing strips of 0/16/32/64/128 rows per chunk: small_grid lines
for s in 0 16 32 64 128; do
  for k in 1 2; do
    timeout 300 python bench.py --steps 5 --warmup 3 --e2e-runs 0 --no-c4 --ooc-gib 0 --matmul-n 0 --no-cpu-baseline --rows 8192 --cols 8192 --c1-strip $s 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read())['small_grid']; print($s, round(d['ms_per_iter']*1e3,2), 'us/iter', round(d['roofline']['frac'],3), d['graph_replays'], d['plan_cache_hits'])"
  done
done
