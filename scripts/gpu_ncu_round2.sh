#!/bin/bash
# Round-2 ncu evidence (numbers printed under ncu are never bench values):
#  * launch list of a short default-size bench run (heat2d 65536^2 at N=1): per-launch times
#  * ncu --set full of the bench's heat2d kernel (65536^2, DRAM traffic for roofline.traffic),
#    the centred-tier k-means assign kernel, the TF32 rounding pass + TF32 GEMM at 16384^3,
#    and the inter-process fused send/recv kernels are covered by the halo trace instead
mkdir -p gpurun_out/ncu2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu2/bench_launches.csv \
  python bench.py --steps 2 --warmup 1 --e2e-runs 0 --no-c4 --no-c1 --ooc-gib 0 --matmul-n 0 --nbody-n 0 --no-cpu-baseline > gpurun_out/ncu2/bench_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:heat2d_tma -s 3 -c 1 -f -o gpurun_out/ncu2/heat2d_tma \
  python bench.py --steps 2 --warmup 1 --e2e-runs 0 --no-c4 --no-c1 --ooc-gib 0 --matmul-n 0 --nbody-n 0 --no-cpu-baseline > gpurun_out/ncu2/heat2d.log 2>&1
python scripts/ncu_heat_summary.py gpurun_out/ncu2/heat2d_tma.ncu-rep gpurun_out/ncu2/heat2d_tma_ncu_summary.json 65536 65536 \
  "ncu --set full -k regex:heat2d_tma -s 3 -c 1 python bench.py --steps 2 --warmup 1 ..." > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmeans_assign_fast -c 1 -f -o gpurun_out/ncu2/kmeans_assign_centred \
  python scripts/km_assign_perf.py 200000000 > gpurun_out/ncu2/km.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm|round_rows" -c 3 -f -o gpurun_out/ncu2/tf32_16384 \
  python scripts/gemm_tf32_perf.py 16384 > gpurun_out/ncu2/tf32.log 2>&1
for f in gpurun_out/ncu2/*.ncu-rep; do echo "== $f"; python scripts/ncu_summary.py $f; done > gpurun_out/ncu2/summary.txt 2>&1
ls -la gpurun_out/ncu2
