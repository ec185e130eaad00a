#!/bin/bash
# world sizes 4 and 8 of the one-process-per-GPU bench path with all ranks sharing one B200
# (gloo for the timing reductions): the inter-process halo messages with interior ranks that
# talk to two neighbours, ring wrap-around over many steps, per-rank e2e boxes
mkdir -p gpurun_out/mr
for n in 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --steps 40 --warmup 3 \
    --rows 8192 --cols 8192 --e2e-runs 1 --e2e-pipeline 4 --e2e-iters 5 > gpurun_out/mr/bench_n$n.json 2> gpurun_out/mr/bench_n$n.err; echo n=$n rc=$?
  tail -2 gpurun_out/mr/bench_n$n.err; cut -c1-300 gpurun_out/mr/bench_n$n.json
done
timeout 600 python -m pytest tests/test_gpu_multiproc.py -q 2>&1 | tail -2
