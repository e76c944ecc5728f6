#!/bin/bash
# weighted SVM chain + inline division: tests, benches, ncu of the weighted kernel
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_division.py tests/test_gpu_chain.py tests/test_gpu_api.py -x -q > gpurun_out/pytest_chain.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_chain.log
bash tools/quickbench.sh svm1m svm1m_rho2 svm1m_w
ncu --set full --clock-control none --import-source on -k "regex:k_svm_chain_w" -s 2 -c 1 \
    -o gpurun_out/r02_chain_w -f python bench.py --workload svm1m_w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_chain_w.log 2>&1; echo "ncu chain_w rc=$?"
