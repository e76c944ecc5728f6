#!/bin/bash
# svm1m / pack5000 / mpc100k bench lines without the CPU baseline (under gpurun)
for w in svm1m pack5000 mpc100k; do
  timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/q3_$w.json 2>gpurun_out/q3_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/q3_$w.json'))
print('$w', round(d['ms_per_step'],4), '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], {k: round(v['ms_avg'],4) for k,v in d['kernels'].items()})"
done
