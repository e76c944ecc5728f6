#!/bin/bash
# weighted SVM chain + MPC inline z division: tests and benches
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_division.py tests/test_gpu_chain.py tests/test_gpu_mpc_block.py -x -q > gpurun_out/pytest_chain.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_chain.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mpc" > gpurun_out/pytest_mpc.log 2>&1; echo "pytest mpc rc=$?"; tail -2 gpurun_out/pytest_mpc.log
bash tools/quickbench.sh svm1m_rho2 svm1m_w mpc100k
FGADMM_MPC_BLOCK=0 timeout 300 python bench.py --workload mpc100k --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mpc_noblock.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_mpc_noblock.json')); print('mpc noblock', d['value'], d['ms_per_step'], {k:round(v['ms_avg'],4) for k,v in d['kernels'].items()})"
