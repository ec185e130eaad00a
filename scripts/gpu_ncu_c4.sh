#!/bin/bash
# ncu --set full captures of the C4 kernels (k-means assign/update, 65536-bin histogram)
mkdir -p gpurun_out
for k in kmeans_update_fast kmeans_assign_fast histogram_pair; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/$k \
    python scripts/c4_perf.py --hist-n 1000000000 --km-n 200000000 --steps 1 > gpurun_out/$k.log 2>&1
done
