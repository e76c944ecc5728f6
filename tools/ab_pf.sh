#!/bin/bash
# A/B of the unit chain: cp.async prefetch buffer vs register loads (under gpurun)
for rep in 1 2; do
for v in pf0 pf1; do
  export FGADMM_CHAIN_PF=${v#pf}
  timeout 300 python bench.py --workload svm1m --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ab_pf_$v.json 2>gpurun_out/ab_pf_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_pf_$v.json'))
print('$v', round(d['ms_per_step'],4), '%.3e'%d['value'], {k: round(v['ms_avg'],4) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
done
