# A/B of the GEMM variants (CTA pair vs single CTA) at a given size and iteration count
SZ=${1:-32768}; IT=${2:-5}
for r in 1 2; do
  timeout 100 python scripts/gemm_sweep.py $SZ $IT
  MTB_GEMM_NO_PAIR=1 timeout 100 python scripts/gemm_sweep.py $SZ $IT
done
