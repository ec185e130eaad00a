#!/bin/bash
# C1 grid (4096^2, 100 iterations, bench leg protocol) with 1, 2, 4 and 8 chunks on one GPU: the
# cost of the halo copies and of splitting the kernel
for f in 0 1; do for c in 1 4 8; do
  for rep in 1 2; do
    echo -n "nofusion=$f chunks $c: "
    MTB_NO_HALO_FUSION=$f timeout 300 python -c "
import bench
d = bench.run_c1(100, 0, 6463.7, False, chunks=$c)
print(round(d['ms_per_iter'] * 1e3, 2), 'us/iter', round(d['roofline']['frac'], 3), d['graph_replays'], 'fused', d['fused_halo_copies'], 'copies', d['halo_copies'])"
  done
done
done
