#!/bin/bash
# A/B the packing kernel variants (under gpurun)
for cv in tile_reg tile generic; do
  for cl in 0 1; do
    if [ $cl = 1 ]; then export FGADMM_NO_CLUSTER=1; else unset FGADMM_NO_CLUSTER; fi
    export FGADMM_COLLISION=$cv
    timeout 300 python bench.py --workload pack5000 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${cv}_${cl}.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab_${cv}_${cl}.json'))
print('$cv nocluster=$cl', round(d['ms_per_step'],3), {k: round(v['ms_avg'],3) for k,v in d['kernels'].items()})"
  done
done
