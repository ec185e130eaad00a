#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over small GPU parity cases: heat2d (TMA and
# register kernels, halo exchange), histogram / k-means reduce trees and the FP32 k-means tier,
# bundled scenarios, ragged grids, the tcgen05 GEMM, gather fuzz, nbody, graph replay, disk tier
mkdir -p gpurun_out/sanitizer
SEL="tests/test_gpu_parity.py::test_heat2d_matches_reference_golden tests/test_gpu_parity.py::test_histogram_matches_reference_golden tests/test_gpu_parity.py::test_kmeans_i32_matches_reference_golden tests/test_gpu_parity.py::test_bundled_scenario_matches_reference tests/test_gpu_edges.py::test_heat2d_ragged_shapes tests/test_gpu_matmul.py::test_matmul_nt_bf16_through_the_planner tests/test_gpu_fuzz.py::test_correlator_like_scenario tests/test_gpu_nbody.py tests/test_gpu_graphs.py::test_replay_interleaved_with_other_work tests/test_gpu_spill.py::test_disk_tier_below_the_host_tier tests/test_gpu_c4.py::test_kmeans_assign_signed_values tests/test_gpu_halo_fusion.py"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all --print-limit 20 \
    python -m pytest $SEL -q -m gpu -p no:cacheprovider -x > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitizer/$tool.log | tail -3
done
MTB_HEAT_TMA=0 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests/test_gpu_edges.py::test_heat2d_ragged_shapes -q -m gpu -p no:cacheprovider > gpurun_out/sanitizer/memcheck_register_heat.log 2>&1
echo "memcheck (register heat2d) rc=$?"; tail -2 gpurun_out/sanitizer/memcheck_register_heat.log
