#!/bin/bash
# full GPU suite + quick benches of the three workloads (under gpurun)
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f_smoke.log
bash tools/quickbench.sh ${QB:-svm1m pack5000 mpc100k svm1m_rho2}
