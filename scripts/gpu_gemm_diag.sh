#!/bin/bash
# DRAM bytes and duration of one 32768^3 launch: single-CTA kernel, CTA-pair kernel, and the
# pair kernel with its C stores skipped (is the extra DRAM read traffic caused by the epilogue?)
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct"
for cfg in "single:MTB_GEMM_NO_PAIR=1" "pair:MTB_GEMM_FORCE_PAIR=1" "pair_nostore:MTB_GEMM_FORCE_PAIR=1 MTB_GEMM_NOSTORE=1" "single_g8:MTB_GEMM_NO_PAIR=1 MTB_GEMM_GROUP=8" "pair_g4:MTB_GEMM_FORCE_PAIR=1 MTB_GEMM_GROUP=4"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_bf16 -c 1 --csv python scripts/gemm_one.py 32768 2>/dev/null | grep -E "gemm_bf16" | awk -F'","' -v n=$name '{print n, $(NF-2), $NF}'
done
