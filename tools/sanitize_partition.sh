#!/bin/bash
export PYTHONFAULTHANDLER=1
for tool in memcheck racecheck; do
timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 10 \
  python -m pytest -x -q tests/test_gpu_partition.py tests/test_gpu_api.py \
  "tests/test_gpu_parity.py::test_mpc_dynamics_forms_match_oracle" "tests/test_gpu_parity.py::test_mpc_16x4_matches_reference" \
  > gpurun_out/${tool}4.log 2>&1
echo "$tool rc=$?"; grep -E "SUMMARY|passed|failed" gpurun_out/${tool}4.log | head -4
grep -A1 "Potential\|Race reported\|Invalid" gpurun_out/${tool}4.log | grep "at " | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head
done
