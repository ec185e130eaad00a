#!/bin/bash
# Scaling proxy on one B200: the C2 bench at N=1, then N=2 and N=4 ranks sharing the GPU under
# MPS (the ranks' kernels run concurrently, so each rank's half / quarter grid, the halo
# messages, the per-rank planning and the max-over-ranks timing all run as they would on
# separate GPUs, at one GPU's bandwidth). Whole-job cell-updates/s at N ranks / N=1 measures
# what the one-process-per-GPU machinery costs beyond the kernel.
mkdir -p gpurun_out/mps
ARGS="--steps 40 --warmup 5 --e2e-runs 0 --no-cpu-baseline --matmul-n 0 --tf32-steps 0 --no-c4 --no-c1 --nbody-n 0 --ooc-gib 0"
timeout 600 python bench.py $ARGS > gpurun_out/mps/n1.json 2> gpurun_out/mps/n1.err; echo n1 rc=$?
for n in 2 4 8; do
  timeout 900 bash scripts/with_mps.sh python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n \
    bench.py --gpus $n $ARGS > gpurun_out/mps/n$n.json 2> gpurun_out/mps/n$n.err; echo n$n rc=$?
done
python - <<'PY'
import json
v = {}
for n in (1, 2, 4, 8):
    try:
        d = json.loads(open(f"gpurun_out/mps/n{n}.json").read().strip().splitlines()[-1])
        v[n] = d["value"]
        print(n, round(d["value"] / 1e9, 1), "Gcell/s", round(d["ms_per_step"], 3), "ms/step")
    except Exception as e:
        print(n, "failed", e)
for n in (2, 4, 8):
    if n in v and 1 in v:
        print(f"N={n} ranks on one GPU under MPS / N=1: {v[n] / v[1]:.3f}")
PY
