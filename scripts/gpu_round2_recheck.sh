mkdir -p gpurun_out/r2c
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2c/gputests.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/r2c/gputests.log
python -c "import __graft_entry__ as g; g.smoke()"
timeout 1200 python bench.py > gpurun_out/r2c/bench_default.json 2> gpurun_out/r2c/bench_default.err; echo bench rc=$?
tail -3 gpurun_out/r2c/bench_default.err; cut -c1-1500 gpurun_out/r2c/bench_default.json
