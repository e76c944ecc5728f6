#!/bin/bash
# A/B of the fused SVM chain variants (under gpurun)
for v in default occ4 nounit nochain; do
  unset FGADMM_CHAIN_OCC3 FGADMM_CHAIN_OCC4 FGADMM_NO_CHAIN FGADMM_CHAIN_NO_UNIT
  [ $v = occ4 ] && export FGADMM_CHAIN_OCC4=1
  [ $v = nochain ] && export FGADMM_NO_CHAIN=1
  [ $v = nounit ] && export FGADMM_CHAIN_NO_UNIT=1
  timeout 300 python bench.py --workload svm1m --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_chain_$v.json 2>gpurun_out/ab_chain_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_chain_$v.json'))
print('$v', round(d['ms_per_step'],3), '%.3e'%d['value'], {k: round(v['ms_avg'],3) for k,v in d['kernels'].items()})"
done
