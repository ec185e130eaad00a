# Functional check of the N>1 bench path on a single GPU (ranks share it over gloo): N=2 and 4
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multiproc.py tests/test_host_io.py -q -m gpu -p no:cacheprovider 2>&1 | tail -5
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 10 --warmup 3 \
  --rows 16384 --cols 16384 --e2e-iters 10 --e2e-pipeline 4 --e2e-runs 1 --no-cpu-baseline > gpurun_out/multi_$n.json 2> gpurun_out/multi_$n.err; echo rc=$?
tail -3 gpurun_out/multi_$n.err; cat gpurun_out/multi_$n.json
done
timeout 600 python bench.py --steps 20 --warmup 3 --matmul-n 0 --no-c4 --no-cpu-baseline --e2e-runs 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['e2e'])"
