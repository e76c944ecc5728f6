#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over small
# device tests covering every kernel form of the round-2 build (under gpurun),
# then the whole GPU suite
export PYTHONFAULTHANDLER=1
mkdir -p gpurun_out
TESTS=("tests/test_gpu_parity.py::test_packing_class_boundaries_bitwise_vs_oracle"
       "tests/test_gpu_parity.py::test_star_quadratic_giant_bitwise"
       "tests/test_gpu_chain.py::test_chain_bitwise_equals_generic[33-32-7]"
       "tests/test_gpu_chain.py::test_chain_general_weights_bitwise[2.0-1.0]"
       "tests/test_gpu_chain.py::test_chain_general_weights_bitwise[0.5-1.3]"
       "tests/test_gpu_chain.py::test_chain_general_weights_bitwise[0.7-1.3]"
       "tests/test_gpu_chain.py::test_chain_random_edge_weights_bitwise_and_oracle"
       "tests/test_gpu_parity.py::test_mpc_chain_bitwise_equals_per_kind"
       "tests/test_gpu_mpc_block.py::test_blocked_chain_bitwise_equals_per_iteration_chain[40-7]"
       "tests/test_gpu_mpc_block.py::test_blocked_chain_bitwise_equals_per_iteration_chain[300-11]"
       "tests/test_gpu_partition.py::test_local_group_matches_single_plan"
       "tests/test_gpu_upload.py")
for tool in memcheck racecheck synccheck initcheck; do
  extra=""; [ $tool = memcheck ] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 20 \
    python -m pytest -x -q -p no:cacheprovider "${TESTS[@]}" > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san_$tool.log | head -5
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu2.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_gpu2.log
