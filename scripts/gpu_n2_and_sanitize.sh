mkdir -p gpurun_out/n2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 \
  --rows 32768 --cols 32768 --e2e-runs 1 --e2e-pipeline 4 --e2e-iters 5 > gpurun_out/n2/bench_n2.json 2> gpurun_out/n2/bench_n2.err; echo n2 rc=$?
tail -3 gpurun_out/n2/bench_n2.err; cut -c1-400 gpurun_out/n2/bench_n2.json
bash scripts/gpu_sanitize.sh
