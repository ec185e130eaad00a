#!/bin/bash
# CTA-pair GEMM with per-CTA (cta_group::1) TMA loads and a relay barrier vs the cta_group::2 loads
M="gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct"
export MTB_GEMM_RELAY=1
timeout 120 python -m pytest tests/test_gpu_matmul.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
for n in 16384 32768; do
  timeout 120 ncu --metrics $M --clock-control none -k regex:gemm_bf16 -c 1 --csv python scripts/gemm_one.py $n 2>/dev/null | grep -E "gemm_bf16" | awk -F'","' -v n=relay_$n '{print n, $(NF-2), $NF}'
done
timeout 300 python scripts/gemm_perf.py 2>&1 | tail -4
