#!/bin/bash
# class-L row stage forms on pack5000 (under gpurun)
for rep in 1 2; do
for v in default deep big; do
  unset FGADMM_PIPE_DEEP FGADMM_PIPE_BIG
  [ $v = deep ] && export FGADMM_PIPE_DEEP=1
  [ $v = big ] && export FGADMM_PIPE_BIG=1
  timeout 300 python bench.py --workload pack5000 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_pipe_$v.json 2>gpurun_out/ab_pipe_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_pipe_$v.json'))
print('$v', round(d['ms_per_step'],4), '%.3e'%d['value'], {k: round(v['ms_avg'],4) for k,v in d['kernels'].items()})"
done
done
