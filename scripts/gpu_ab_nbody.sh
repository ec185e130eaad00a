#!/bin/bash
# n-body A/B on one B200: bodies per CTA (MTB_NB_THREADS) x pair-group width (MTB_NB_UNROLL),
# the bit-exact tests first, then one ncu --set full capture of the default kernel.
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests/test_gpu_nbody.py -x -q 2>&1 | tail -3
for t in 128 64 32; do for u in 4 2; do MTB_NB_THREADS=$t MTB_NB_UNROLL=$u timeout 300 python scripts/nbody_perf.py 65536 | sed "s/^/T=$t U=$u /"; done; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:nbody_tiled -c 1 -o gpurun_out/ab/nbody_full -f python scripts/nbody_perf.py 65536 > gpurun_out/ab/ncu.log 2>&1; echo ncu rc=$?
