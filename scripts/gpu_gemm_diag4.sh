#!/bin/bash
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct"
for cfg in "pair_sync:MTB_GEMM_FORCE_PAIR=1 MTB_GEMM_START_SYNC=1" "pair_sync_16k:MTB_GEMM_START_SYNC=1"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  n=32768; [ "$name" = "pair_sync_16k" ] && n=16384
  env $envs timeout 120 ncu --metrics $M --clock-control none -k regex:gemm_bf16 -c 1 --csv python scripts/gemm_one.py $n 2>/dev/null | grep -E "gemm_bf16" | awk -F'","' -v n=$name '{print n, $(NF-2), $NF}'
done
