#!/bin/bash
# Round-2 check on one B200: FFMA probe, the N=2 bench path (two ranks share the GPU: gloo for
# the timing reductions), then the default bench line and the reference arm.
mkdir -p gpurun_out/r2
python -c "
import ctypes; l = ctypes.CDLL('scripts/microbench/libfma_probe.so'); l.mt_probe_ffma_dot.restype = ctypes.c_double
print('ffma dot probe', l.mt_probe_ffma_dot(20), 'Tmac/s')"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 \
  --rows 32768 --cols 32768 --e2e-runs 1 --e2e-pipeline 4 --e2e-iters 5 > gpurun_out/r2/bench_n2.json 2> gpurun_out/r2/bench_n2.err; echo n2 rc=$?
tail -3 gpurun_out/r2/bench_n2.err; cut -c1-600 gpurun_out/r2/bench_n2.json
timeout 1200 python bench.py > gpurun_out/r2/bench_default.json 2> gpurun_out/r2/bench_default.err; echo bench rc=$?
tail -3 gpurun_out/r2/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/r2/bench_ref.json 2> gpurun_out/r2/bench_ref.err; echo ref rc=$?
cat gpurun_out/r2/bench_ref.json | cut -c1-300
