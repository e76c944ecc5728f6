#!/bin/bash
# racecheck of the MPC chain / block kernels, then the mpc100k quick bench
export PYTHONFAULTHANDLER=1
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q -p no:cacheprovider "tests/test_gpu_mpc_block.py::test_blocked_chain_bitwise_equals_per_iteration_chain[40-7]" "tests/test_gpu_mpc_block.py::test_blocked_chain_bitwise_equals_per_iteration_chain[300-11]" "tests/test_gpu_parity.py::test_mpc_chain_bitwise_equals_per_kind" > gpurun_out/san_race_mpc.log 2>&1
echo "racecheck rc=$?"; grep -E "SUMMARY|passed|failed" gpurun_out/san_race_mpc.log | head -5
bash tools/quickbench.sh mpc100k
