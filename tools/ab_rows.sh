#!/bin/bash
for v in r512 r256; do
  unset FGADMM_ROW256
  [ $v = r256 ] && export FGADMM_ROW256=1
  timeout 300 python bench.py --workload pack5000 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_rows_$v.json 2>gpurun_out/ab_rows_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_rows_$v.json'))
print('$v', round(d['ms_per_step'],4), '%.3e'%d['value'], {k: round(v['ms_avg'],4) for k,v in d['kernels'].items()})"
done
