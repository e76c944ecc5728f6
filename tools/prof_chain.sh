#!/bin/bash
# packing gpu tests (collision v3) + ncu of the chain kernel and collision v3
timeout 900 python -m pytest tests -m gpu -x -q -k "packing or chain or collision or opt_in" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
bash tools/quickbench.sh pack5000 svm1m
ncu --set full --clock-control none --import-source on -k "regex:k_svm_chain" -s 2 -c 1 \
    -o gpurun_out/full_chain -f python bench.py --workload svm1m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/full_chain.log 2>&1
echo "ncu chain rc=$?"
ncu --set full --clock-control none --import-source on -k "regex:k_collision_tiles_v3|k_var_large_vec" -s 3 -c 3 \
    -o gpurun_out/full_pack_v3 -f python bench.py --workload pack5000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/full_pack_v3.log 2>&1
echo "ncu pack rc=$?"
