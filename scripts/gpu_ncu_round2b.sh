#!/bin/bash
# Round-2 (second session) ncu evidence; numbers printed under ncu are never bench values.
#  * ncu --set full of the wide CTA-pair contraction at 32768^3 (the bench's C3 kernel)
#  * C1 (4096^2, 4 chunks, fused halos, L2-resident steps): per-launch duration and DRAM bytes of
#    the heat2d kernels and every other kernel of a short C1 run
mkdir -p gpurun_out/ncu3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_nt_2sm -c 1 -f -o gpurun_out/ncu3/gemm_wide_32768 \
  python scripts/gemm_one.py 32768 > gpurun_out/ncu3/gemm.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu3/gemm_wide_32768.ncu-rep > gpurun_out/ncu3/gemm_wide_32768_summary.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/ncu3/c1_launches.csv python -c "
import bench
print(bench.run_c1(20, 0, 6463.7, False))" > gpurun_out/ncu3/c1.log 2>&1
python - <<'PY' > gpurun_out/ncu3/c1_launches_summary.txt
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/ncu3/c1_launches.csv")) if len(r) > 10 and r[0].isdigit()]
per = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    per[r[4][:60]][r[12]].append(float(r[14]))
for k, m in per.items():
    n = len(m["gpu__time_duration.sum"])
    t = sum(m["gpu__time_duration.sum"]) / max(1, n) / 1e3
    rd = sum(m["dram__bytes_read.sum"]) / max(1, n) / 1e6
    wr = sum(m["dram__bytes_write.sum"]) / max(1, n) / 1e6
    print(f"{k:60s} launches {n:4d} mean {t:8.2f} us  DRAM read {rd:8.2f} MB write {wr:8.2f} MB per launch")
PY
cat gpurun_out/ncu3/c1_launches_summary.txt gpurun_out/ncu3/gemm_wide_32768_summary.txt
ls -la gpurun_out/ncu3
