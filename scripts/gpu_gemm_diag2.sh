#!/bin/bash
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct"
for cfg in "pair_nmajor16:MTB_GEMM_FORCE_PAIR=1 MTB_GEMM_NMAJOR=1" "pair_nmajor4:MTB_GEMM_FORCE_PAIR=1 MTB_GEMM_NMAJOR=1 MTB_GEMM_GROUP=4" "pair_evl:MTB_GEMM_FORCE_PAIR=1 MTB_GEMM_HINT_A=14F0000000000000 MTB_GEMM_HINT_B=14F0000000000000" "pair_cl32:MTB_GEMM_FORCE_PAIR=1 MTB_GEMM_CLUSTERS=32" "pair_16k:MTB_GEMM_FORCE_PAIR=1"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  n=32768; [ "$name" = "pair_16k" ] && n=16384
  env $envs timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_bf16 -c 1 --csv python scripts/gemm_one.py $n 2>/dev/null | grep -E "gemm_bf16" | awk -F'","' -v n=$name '{print n, $(NF-2), $NF}'
done
