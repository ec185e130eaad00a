#!/bin/bash
# A/B on one B200: n-body pair-group width (MTB_NB_UNROLL) and k-means grouped-maximum variants
# (MTB_KM_VARIANT; the sha256 of the assignments must agree across variants).
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests/test_gpu_nbody.py tests/test_gpu_c4.py -x -q 2>&1 | tail -3
for u in 4 2 8; do MTB_NB_UNROLL=$u timeout 300 python scripts/nbody_perf.py 65536 | sed "s/^/U=$u /"; done
for v in 0 6 7 8 0 6; do MTB_KM_VARIANT=$v timeout 300 python scripts/km_assign_perf.py; done
