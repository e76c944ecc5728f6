#!/bin/bash
# A/B: in-tree build vs build_ab/lib_head.so on the listed workloads (QB)
set -u
for rep in 1 2 3; do
  bash tools/quickbench.sh ${QB} 2>&1 | grep -A1 "EU/s" | sed "s/^/[new] /"
  FGADMM_LIB=$PWD/build_ab/lib_head.so bash tools/quickbench.sh ${QB} 2>&1 | grep -A1 "EU/s" | sed "s/^/[old] /"
done
