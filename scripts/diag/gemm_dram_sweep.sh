#!/bin/bash
# 32768^3 bf16 contraction: DRAM bytes, L2 hit rate and duration of one launch (ncu, cold
# cache) per kernel / schedule / rasterisation group, then event timings of the same variants
# (best and median of 5 launches after 2 warm-ups).
#   usage: scripts/diag/gemm_dram_sweep.sh [n] [variants...]
#   variant = single-static | single-dyn-G | pair-static-G | pair-dyn-G | wide-static-G | wide-dyn-G
mkdir -p gpurun_out
n=${1:-32768}; shift
variants=${@:-"single-static pair-dyn-4 pair-dyn-8 pair-dyn-16"}
envs_of() {
  case $1 in
    single-static) echo "MTB_GEMM_NO_PAIR=1" ;;
    single-dyn-*) echo "MTB_GEMM_NO_PAIR=1 MTB_GEMM_DYNAMIC=1 MTB_GEMM_GROUP=${1##*-}" ;;
    pair-static-*) echo "MTB_GEMM_FORCE_PAIR=1 MTB_GEMM_WIDE=0 MTB_GEMM_GROUP=${1##*-}" ;;
    pair-dyn-*) echo "MTB_GEMM_FORCE_PAIR=1 MTB_GEMM_WIDE=0 MTB_GEMM_DYNAMIC=1 MTB_GEMM_GROUP=${1##*-}" ;;
    wide-dyn-*) echo "MTB_GEMM_WIDE=1 MTB_GEMM_DYNAMIC=1 MTB_GEMM_GROUP=${1##*-}" ;;
    wide-static-*) echo "MTB_GEMM_WIDE=1 MTB_GEMM_STATIC=1 MTB_GEMM_GROUP=${1##*-}" ;;
    *) echo "unknown variant $1" >&2; exit 1 ;;
  esac
}
for v in $variants; do
  env $(envs_of $v) timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_op_gemm_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:gemm -c 1 --csv python scripts/gemm_one.py $n 2>/dev/null | grep -E '"(dram__|gpu__time|lts__|sm__pipe)' \
    | awk -F'","' -v v=$v '{printf "%s %s %s %s\n", v, $(NF-2), $(NF-1), $NF}' | tr -d '"'
done
for v in $variants; do
  echo -n "$v: "
  env $(envs_of $v) timeout 600 python scripts/gemm_perf_one.py $n
done
