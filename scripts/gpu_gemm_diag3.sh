#!/bin/bash
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct"
for cfg in "pair_nohint:MTB_GEMM_FORCE_PAIR=1 MTB_GEMM_HINT_A=0 MTB_GEMM_HINT_B=0" "pair_nohint_16k:MTB_GEMM_HINT_A=0 MTB_GEMM_HINT_B=0"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  n=32768; [ "$name" = "pair_nohint_16k" ] && n=16384
  env $envs timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_bf16 -c 1 --csv python scripts/gemm_one.py $n 2>/dev/null | grep -E "gemm_bf16" | awk -F'","' -v n=$name '{print n, $(NF-2), $NF}'
done
