#!/bin/bash
# DRAM bytes of one 32768^3 bf16 contraction launch per scheduling variant (ncu, cold cache)
mkdir -p gpurun_out
for v in static dynamic; do
  extra=""; [ $v = static ] && extra="MTB_GEMM_STATIC=1"
  env MTB_GEMM_FORCE_PAIR=1 $extra timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:gemm -c 1 --csv python scripts/gemm_sched_ab.py 32768 2>/dev/null | grep -E "dram__|gpu__time|lts__" | sed "s/^/$v: /" | cut -c1-40,150-
done
