#!/bin/bash
ncu --set full --clock-control none --import-source on -k "regex:k_var_giant_chunks" -s 2 -c 1 \
    -o gpurun_out/gchunks -f python bench.py --workload svm1m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gchunks_ncu.log 2>&1
echo "ncu rc=$?"
FGADMM_GIANT_UNFUSED=1 ncu --set full --clock-control none --import-source on -k "regex:k_var_giant_chunks" -s 2 -c 1 \
    -o gpurun_out/gchunks_unf -f python bench.py --workload svm1m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gchunks_unf_ncu.log 2>&1
echo "ncu rc=$?"
