#!/bin/bash
# class-L rows: phase 2 through the ring vs straight from L2 (under gpurun)
for rep in 1 2; do
for v in default d2only ringall; do
  unset FGADMM_ROW_RING FGADMM_ROW_DIRECT2
  [ $v = d2only ] && export FGADMM_ROW_DIRECT2=1
  [ $v = ringall ] && export FGADMM_ROW_DIRECT2=1 FGADMM_ROW_RING=1
  timeout 300 python bench.py --workload pack5000 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_d2_$v.json 2>gpurun_out/ab_d2_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_d2_$v.json'))
print('$v', round(d['ms_per_step'],4), '%.3e'%d['value'], {k: round(v['ms_avg'],4) for k,v in d['kernels'].items()})"
done
done
