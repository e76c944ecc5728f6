#!/bin/bash
export PYTHONFAULTHANDLER=1
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q tests/test_gpu_parity.py -k "opt_in" > gpurun_out/racecheck2.log 2>&1
echo "racecheck opt_in rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed|Race" gpurun_out/racecheck2.log | head -8
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest -x -q tests/test_gpu_parity.py -k "opt_in" > gpurun_out/memcheck2.log 2>&1
echo "memcheck opt_in rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid" gpurun_out/memcheck2.log | head -8
