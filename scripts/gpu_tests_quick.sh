#!/bin/bash
# GPU test suite + smoke on one B200 (log under gpurun_out/tests/).
mkdir -p gpurun_out/tests
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/tests/gputests.log 2>&1; echo tests rc=$?; tail -4 gpurun_out/tests/gputests.log
python -c "import __graft_entry__ as g; g.smoke()"
