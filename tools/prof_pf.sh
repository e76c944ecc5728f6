#!/bin/bash
for v in 0 1; do
  FGADMM_CHAIN_PF=$v ncu --set full --clock-control none --import-source on -k "regex:k_svm_chain_unit" -s 2 -c 1 \
    -o gpurun_out/pf$v -f python bench.py --workload svm1m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pf$v.log 2>&1
  echo "ncu pf$v rc=$?"
done
