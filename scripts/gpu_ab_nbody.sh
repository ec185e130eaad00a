#!/bin/bash
# n-body on one B200: bit-exact tests, then the n = 65536 step (nbody_perf.py) and one ncu capture
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests/test_gpu_nbody.py -x -q 2>&1 | tail -1
for rep in 1 2 3; do timeout 300 python scripts/nbody_perf.py 65536; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:nbody_tiled -c 1 -o gpurun_out/ab/nbody_full -f python scripts/nbody_perf.py 65536 > gpurun_out/ab/ncu.log 2>&1; echo ncu rc=$?
