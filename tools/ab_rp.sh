#!/bin/bash
for rep in 1 2; do
for v in def rp; do
  unset FGADMM_CHAIN_RP
  [ $v = rp ] && export FGADMM_CHAIN_RP=1
  timeout 300 python bench.py --workload svm1m --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ab_rp_$v.json 2>gpurun_out/ab_rp_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_rp_$v.json'))
print('$v', round(d['ms_per_step'],4), '%.3e'%d['value'], {k: round(v['ms_avg'],4) for k,v in d['kernels'].items()})"
done
done
