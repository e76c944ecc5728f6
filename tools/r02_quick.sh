#!/bin/bash
# quick round-2 iteration: chain tests, NCCL test details, benches, MPC block ncu
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_nccl.py -x -q -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/q_pytest.log | tail -15
bash tools/quickbench.sh ${QB:-svm1m svm1m_rho2 svm1m_w}
if [ "${PROF_MPC:-1}" = 1 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_mpc_block$" -s 1 -c 1 \
      -o gpurun_out/q_mpcblock -f python bench.py --workload mpc100k --steps 12 --warmup 3 --no-cpu-baseline \
      > gpurun_out/q_mpcblock.log 2>&1
  echo "ncu mpc rc=$?"
  ncu -i gpurun_out/q_mpcblock.ncu-rep --page raw --csv > gpurun_out/q_mpcblock_raw.csv 2>/dev/null
  ncu -i gpurun_out/q_mpcblock.ncu-rep --page details --csv > gpurun_out/q_mpcblock_details.csv 2>/dev/null
  ncu -i gpurun_out/q_mpcblock.ncu-rep --page source --csv --print-source sass > gpurun_out/q_mpcblock_sass.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/q_mpcblock.ncu-rep > gpurun_out/q_mpcblock.md 2>&1
  rm -f gpurun_out/q_mpcblock.ncu-rep
fi
du -sh gpurun_out
