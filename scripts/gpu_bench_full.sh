#!/bin/bash
# Full default bench line + reference arm on one B200 (profiles/round2/bench_full.json)
mkdir -p gpurun_out/full
timeout 1500 python bench.py > gpurun_out/full/bench.json 2> gpurun_out/full/bench.err; echo bench rc=$?
tail -3 gpurun_out/full/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/full/bench_ref.json 2> gpurun_out/full/bench_ref.err; echo ref rc=$?
cut -c1-300 gpurun_out/full/bench_ref.json
