#!/bin/bash
export PYTHONFAULTHANDLER=1
for tool in racecheck synccheck initcheck; do
timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q "tests/test_gpu_parity.py::test_packing_class_boundaries_bitwise_vs_oracle" \
  "tests/test_gpu_parity.py::test_star_quadratic_giant_bitwise" \
  "tests/test_gpu_chain.py::test_chain_bitwise_equals_generic[33-32-7]" \
  "tests/test_gpu_parity.py::test_mpc_chain_bitwise_equals_per_kind" \
  > gpurun_out/$tool.log 2>&1
echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/$tool.log | head -5
done
