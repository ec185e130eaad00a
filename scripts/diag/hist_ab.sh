#!/bin/bash
# 65536-bin histogram A/B: loads in flight per thread (MTB_HIST_U 2 / 4); histogram parity tests first
timeout 900 python -m pytest tests/test_gpu_c4.py tests/test_gpu_parity.py -q -x -k "hist" 2>&1 | tail -1
MTB_HIST_U=4 timeout 900 python -m pytest tests/test_gpu_c4.py -q -x -k "hist" 2>&1 | tail -1
for rep in 1 2; do for u in 2 4; do MTB_HIST_U=$u timeout 300 python scripts/c4_perf.py --hist-n 4000000000 --km-n 0 --steps 10 2>&1 | grep 65536 | sed "s/^/U=$u /"; done; done
