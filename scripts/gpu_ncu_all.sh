#!/bin/bash
# ncu --set full captures of the C4 kernels and nbody_like, plus a launch list of the C4 steps
# (numbers printed under ncu are never bench values)
mkdir -p gpurun_out/ncu
for k in kmeans_update_fast kmeans_assign_fast histogram_pair; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/ncu/$k \
    python scripts/c4_perf.py --hist-n 1000000000 --km-n 200000000 --steps 1 > gpurun_out/ncu/$k.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/c4_launches.csv \
  python scripts/c4_perf.py --hist-n 1000000000 --km-n 200000000 --steps 2 > gpurun_out/ncu/c4_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nbody -c 1 -f -o gpurun_out/ncu/nbody \
  python scripts/nbody_perf.py 32768 > gpurun_out/ncu/nbody.log 2>&1
for f in gpurun_out/ncu/*.ncu-rep; do python scripts/ncu_summary.py $f; done > gpurun_out/ncu/summary.txt 2>&1
ls -la gpurun_out/ncu
