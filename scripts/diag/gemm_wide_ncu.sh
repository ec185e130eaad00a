#!/bin/bash
# ncu --set full of the wide CTA-pair contraction at 32768^3 (one cold launch) with the transposed
# epilogue, and the per-row epilogue (MTB_GEMM_EPI=0) for comparison
mkdir -p gpurun_out/ncu4
for e in 1 0; do
  MTB_GEMM_EPI=$e timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_nt_2sm -c 1 -f -o gpurun_out/ncu4/gemm_wide_32768_epi$e \
    python scripts/gemm_one.py 32768 > gpurun_out/ncu4/gemm_epi$e.log 2>&1; echo epi=$e rc=$?
  python scripts/ncu_summary.py gpurun_out/ncu4/gemm_wide_32768_epi$e.ncu-rep > gpurun_out/ncu4/gemm_wide_32768_epi${e}_summary.txt 2>&1
done
cat gpurun_out/ncu4/*_summary.txt
