#!/bin/bash
# ncu --set full of the 65536-bin histogram kernel (u8 counters, two CTAs per SM) at n = 4e9
mkdir -p gpurun_out/hist
timeout 900 ncu --set full --import-source on --clock-control none -k regex:histogram_quad -c 1 -o gpurun_out/hist/hist65536_full -f \
  python scripts/c4_perf.py --hist-n 4000000000 --km-n 0 --steps 1 > gpurun_out/hist/ncu.log 2>&1; echo ncu rc=$?
