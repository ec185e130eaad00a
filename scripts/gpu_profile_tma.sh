#!/bin/bash
# ncu evidence for the bench's top kernel (TMA-staged heat2d, one GPU). Numbers printed under ncu
# are never bench values.
mkdir -p gpurun_out/prof
CMD="python bench.py --steps 4 --warmup 2 --e2e-runs 0 --no-cpu-baseline --matmul-n 0 --no-c4 --no-c1 --ooc-gib 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/heat2d_tma_launches.csv $CMD > gpurun_out/prof/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:heat2d_tma -s 3 -c 1 -f -o gpurun_out/prof/heat2d_tma_full $CMD > gpurun_out/prof/full.log 2>&1
python scripts/ncu_heat_summary.py gpurun_out/prof/heat2d_tma_full.ncu-rep gpurun_out/prof/heat2d_tma_ncu_summary.json 65536 65536 \
  "ncu --set full --clock-control none --import-source on -k regex:heat2d_tma -s 3 -c 1 $CMD"
