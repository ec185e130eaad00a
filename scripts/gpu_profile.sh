# ncu evidence for the bench's top kernel (one GPU). Numbers printed under ncu are never bench values.
set -x
CMD="python bench.py --steps 4 --warmup 2 --e2e-runs 0 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/launches_bench.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:heat2d_tma -s 3 -c 1 -o gpurun_out/heat2d_full $CMD > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
