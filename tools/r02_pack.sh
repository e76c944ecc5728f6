#!/bin/bash
# packing iteration: bitwise tests and the pack5000 bench
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "packing" -x -q -p no:cacheprovider > gpurun_out/p_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/p_pytest.log
timeout 900 python -m pytest tests/test_gpu_scale.py::test_pack5000_10_iterations_bitwise_vs_oracle tests/test_gpu_convergence.py -x -q -p no:cacheprovider > gpurun_out/p_pytest2.log 2>&1
echo "pytest2 rc=$?"; tail -2 gpurun_out/p_pytest2.log
bash tools/quickbench.sh pack5000 pack5000
