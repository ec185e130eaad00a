mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:heat2d -c 60 --csv --log-file gpurun_out/c1_launches.csv python bench.py --steps 2 --warmup 1 --e2e-runs 0 --no-c4 --ooc-gib 0 --matmul-n 0 --no-cpu-baseline --rows 4096 --cols 4096 > /dev/null 2>&1
tail -5 gpurun_out/c1_launches.csv
