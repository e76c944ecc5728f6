#!/bin/bash
# unit chain bench, two repetitions (under gpurun)
for rep in 1 2; do
  timeout 300 python bench.py --workload svm1m --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ab_xi_$rep.json 2>gpurun_out/ab_xi_$rep.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_xi_$rep.json'))
print('rep$rep', round(d['ms_per_step'],4), '%.3e'%d['value'], {k: round(v['ms_avg'],4) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
ncu --set full --clock-control none --import-source on -k "regex:k_svm_chain_unit" -s 2 -c 1 \
    -o gpurun_out/xi -f python bench.py --workload svm1m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/xi_ncu.log 2>&1
echo "ncu rc=$?"
