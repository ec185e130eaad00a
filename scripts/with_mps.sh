#!/bin/bash
# Runs "$@" under an MPS control daemon (so processes sharing the one GPU run concurrently
# instead of time-slicing), then stops the daemon. Directories under /tmp.
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mtb_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mtb_mps_log
mkdir -p "$CUDA_MPS_PIPE_DIRECTORY" "$CUDA_MPS_LOG_DIRECTORY"
nvidia-cuda-mps-control -d || { echo "mps: daemon failed to start"; exit 90; }
sleep 1
"$@"
rc=$?
echo quit | nvidia-cuda-mps-control
sleep 1
exit $rc
