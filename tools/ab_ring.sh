#!/bin/bash
# A/B of the persistent class-L row ring vs one CTA per row (under gpurun)
for rep in 1 2; do
for v in ring0 ring1 ring1small; do
  unset FGADMM_ROW_RING FGADMM_PIPE_BIG
  [ $v = ring0 ] && export FGADMM_ROW_RING=0
  [ $v = ring1 ] && export FGADMM_ROW_RING=1
  [ $v = ring1small ] && export FGADMM_ROW_RING=1 FGADMM_PIPE_BIG=0
  timeout 300 python bench.py --workload pack5000 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_ring_$v.json 2>gpurun_out/ab_ring_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_ring_$v.json'))
print('$v', round(d['ms_per_step'],4), '%.3e'%d['value'], {k: round(v['ms_avg'],4) for k,v in d['kernels'].items()})"
done
done
