#!/bin/bash
# heat2d TMA kernel L2 residency modes (MTB_HEAT_L2, heat2d.cu) on the C1 grid (4096^2, 4 chunks,
# 100 iterations, graph-batched like the bench leg) and on a 16384^2 x 4-chunk grid
for m in 0 1 2 3; do
  for rep in 1 2; do
    echo -n "mode $m C1: "
    MTB_HEAT_L2=$m timeout 300 python -c "
import bench, json
d = bench.run_c1(100, 0, 6463.7, False)
print(round(d['ms_per_iter'] * 1e3, 2), 'us/iter', round(d['roofline']['frac'], 3))"
  done
  echo -n "mode $m 16384^2x4: "
  MTB_HEAT_L2=$m timeout 300 python scripts/c1_perf.py 16384 4 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_iter']*1e3,1), 'us/iter', 'bound', round(d['hbm_bound_ms_per_iter']*1e3,1))"
done
