#!/bin/bash
# compute-sanitizer memcheck / racecheck over small device tests (under gpurun)
export PYTHONFAULTHANDLER=1
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q tests/test_gpu_upload.py "tests/test_gpu_parity.py::test_packing_100_bit_identical" \
  "tests/test_gpu_parity.py::test_packing_class_boundaries_bitwise_vs_oracle" \
  "tests/test_gpu_parity.py::test_star_quadratic_giant_bitwise" \
  "tests/test_gpu_parity.py::test_mpc_chain_bitwise_equals_per_kind" \
  "tests/test_gpu_chain.py::test_chain_bitwise_equals_generic" \
  > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid" gpurun_out/memcheck.log | head -20
