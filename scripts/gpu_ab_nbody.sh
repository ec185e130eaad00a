#!/bin/bash
# n-body A/B on one B200: one lane per body (default) vs two (MTB_NB_LANES=2), the bit-exact
# tests for both first.
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests/test_gpu_nbody.py -x -q 2>&1 | tail -1
MTB_NB_LANES=2 timeout 600 python -m pytest tests/test_gpu_nbody.py -x -q 2>&1 | tail -1
for rep in 1 2; do for l in 1 2; do MTB_NB_LANES=$l timeout 300 python scripts/nbody_perf.py 65536 | sed "s/^/lanes=$l /"; done; done
MTB_NB_LANES=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:nbody_lanes -c 1 -o gpurun_out/ab/nbody_lanes_full -f python scripts/nbody_perf.py 65536 > gpurun_out/ab/ncu_lanes.log 2>&1; echo ncu rc=$?
