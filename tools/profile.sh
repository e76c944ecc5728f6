#!/bin/bash
# ncu captures for the bench workloads (run under gpurun; 1 GPU).
# usage: tools/profile.sh <workload> <kernel-regex> [count]
set -u
W=$1; K=$2; C=${3:-2}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:$K" -s 4 -c "$C" \
    -o "gpurun_out/prof_${W}" -f \
    python bench.py --workload "$W" --steps 3 --warmup 3 --no-cpu-baseline \
    > "gpurun_out/prof_${W}.log" 2>&1
echo "ncu $W rc=$?"
