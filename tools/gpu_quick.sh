#!/bin/bash
# gpu tests (optionally a subset) + quick benches: tools/gpu_quick.sh "<pytest -k expr>" workloads...
set -u
mkdir -p gpurun_out
K=${1:-}
shift || true
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
fi
echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
bash tools/quickbench.sh "$@"
