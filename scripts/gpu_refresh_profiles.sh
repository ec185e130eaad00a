#!/bin/bash
# refresh ncu evidence for the kernels changed late in the round and the large OOC run
mkdir -p gpurun_out/refresh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kmeans_assign_fast -c 1 -f -o gpurun_out/refresh/kmeans_assign_fp32 \
  python scripts/c4_perf.py --hist-n 1048576 --km-n 200000000 --steps 1 > gpurun_out/refresh/km.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nbody -c 1 -f -o gpurun_out/refresh/nbody_unrolled \
  python scripts/nbody_perf.py 65536 > gpurun_out/refresh/nbody.log 2>&1
python scripts/ncu_summary.py gpurun_out/refresh/kmeans_assign_fp32.ncu-rep gpurun_out/refresh/nbody_unrolled.ncu-rep > gpurun_out/refresh/summary.txt 2>&1
timeout 900 python scripts/ooc_bench.py --rows 327680 --capacity-gib 48 --host-gib 120 --iters 8 > gpurun_out/refresh/ooc_160gib_cap48.json 2> gpurun_out/refresh/ooc.err
cat gpurun_out/refresh/summary.txt; cat gpurun_out/refresh/ooc_160gib_cap48.json
