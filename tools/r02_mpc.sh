#!/bin/bash
# MPC block kernel iteration: bitwise tests, bench, ncu of the block kernel
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mpc_block.py tests/test_gpu_scale.py::test_mpc100k_10_iterations_vs_oracle -x -q -p no:cacheprovider > gpurun_out/m_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/m_pytest.log
bash tools/quickbench.sh mpc100k mpc100k
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_mpc_block$" -s 1 -c 1 \
    -o gpurun_out/m_mpcblock -f python bench.py --workload mpc100k --steps 12 --warmup 3 --no-cpu-baseline \
    > gpurun_out/m_mpcblock.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/m_mpcblock.ncu-rep --page details --csv > gpurun_out/m_mpcblock_details.csv 2>/dev/null
ncu -i gpurun_out/m_mpcblock.ncu-rep --page source --csv --print-source sass > gpurun_out/m_mpcblock_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/m_mpcblock.ncu-rep > gpurun_out/m_mpcblock.md 2>&1
rm -f gpurun_out/m_mpcblock.ncu-rep
cat gpurun_out/m_mpcblock.md
