#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q -k "chain or svm" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
bash tools/ab_chain.sh
ncu --set full --clock-control none --import-source on -k "regex:k_svm_chain_fast" -s 2 -c 1 \
    -o gpurun_out/full_chain2 -f python bench.py --workload svm1m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/full_chain2.log 2>&1
echo "ncu chain rc=$?"
