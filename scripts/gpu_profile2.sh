# ncu captures for the contraction, histogram and k-means kernels (one GPU)
set -x
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 1 -c 1 -o gpurun_out/gemm_full python scripts/gemm_perf.py > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"histogram_smem|histogram_pair|kmeans_assign_fast|kmeans_update_fast" -c 4 -o gpurun_out/c4_full python scripts/c4_perf.py --hist-n 1000000000 --km-n 100000000 --steps 1 > gpurun_out/ncu_c4.log 2>&1
ls -la gpurun_out/*.ncu-rep
