#!/bin/bash
for v in fused unfused; do
  unset FGADMM_GIANT_UNFUSED
  [ $v = unfused ] && export FGADMM_GIANT_UNFUSED=1
  timeout 300 python bench.py --workload svm1m --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ab_g2_$v.json 2>gpurun_out/ab_g2_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_g2_$v.json'))
print('$v', round(d['ms_per_step'],4), '%.3e'%d['value'], {k: round(v['ms_avg'],4) for k,v in d['kernels'].items()})"
done
ncu --set full --clock-control none --import-source on -k "regex:k_var_giant" -s 4 -c 2 \
    -o gpurun_out/giant2 -f python bench.py --workload svm1m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/giant2_ncu.log 2>&1
echo "ncu rc=$?"
