set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
free -g | head -2; nproc
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -40
timeout 600 python bench.py --steps 50 --warmup 5 --e2e-runs 1 --cpu-iters 2 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
