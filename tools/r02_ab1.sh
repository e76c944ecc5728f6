#!/bin/bash
# round 2: weighted SVM chain A/B + ncu of the MPC block and weighted chain kernels
set -u
mkdir -p gpurun_out
bash tools/quickbench.sh svm1m_rho2 svm1m_w
FGADMM_CHAIN_NO_UNIT=1 timeout 600 python bench.py --workload svm1m --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_svm1m_nounit.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_svm1m_nounit.json')); print('nounit', d['value'], d['ms_per_step'], {k:round(v['ms_avg'],4) for k,v in d['kernels'].items()})"
FGADMM_NO_CHAIN=1 timeout 600 python bench.py --workload mpc100k --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mpc_nochain.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_mpc_nochain.json')); print('mpc nochain', d['value'], d['ms_per_step'], {k:round(v['ms_avg'],4) for k,v in d['kernels'].items()})"
ncu --set full --clock-control none --import-source on -k "regex:k_mpc_block" -s 2 -c 1 \
    -o gpurun_out/r02_mpc_block -f python bench.py --workload mpc100k --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_mpc_block.log 2>&1; echo "ncu mpc rc=$?"
ncu --set full --clock-control none --import-source on -k "regex:k_svm_chain" -s 3 -c 1 \
    -o gpurun_out/r02_chain_w -f python bench.py --workload svm1m_w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_chain_w.log 2>&1; echo "ncu chain_w rc=$?"
