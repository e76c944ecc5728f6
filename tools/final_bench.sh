#!/bin/bash
# default bench (svm1m, 50 steps, cpu baseline) + the other workloads + reference arm
set -u
mkdir -p gpurun_out
for w in svm1m pack5000 mpc100k; do
  timeout 900 python bench.py --workload $w > gpurun_out/final_bench_$w.json 2> gpurun_out/final_bench_$w.err
  echo "bench $w rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/final_bench_$w.json'))
print('$w', '%.3e'%d['value'], round(d['ms_per_step'],4), 'e2e %.3e'%d['e2e']['value'], 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'cpu %.3e'%d['cpu_baseline']['value'], d['clocks'])"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"; cat gpurun_out/final_ref.json
