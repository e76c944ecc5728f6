#!/bin/bash
# round 2 evidence (under gpurun, 1 GPU): GPU tests, the default bench
# line, the reference arm at full size, launch lists and ncu --set full
# captures of each workload's top kernels.  The .ncu-rep files are
# summarised on the box (raw CSV + markdown) and removed, so gpurun_out/
# stays under the 64 MiB copy-back limit.  Results in gpurun_out/r02_*.
set -u
mkdir -p gpurun_out
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_gpu.log
fi
timeout 900 python bench.py > gpurun_out/r02_bench_svm1m.json 2> gpurun_out/r02_bench_svm1m.err
echo "bench svm1m rc=$?"; head -c 400 gpurun_out/r02_bench_svm1m.json; echo
if [ "${SKIP_REF:-0}" != 1 ]; then
  timeout 1500 python bench.py --impl reference > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err
  echo "ref rc=$?"; head -c 300 gpurun_out/r02_ref.json; echo
fi
for w in svm1m svm1m_rho2 pack5000 mpc100k; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_$w.csv \
      python bench.py --workload $w --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/r02_launches_$w.log 2>&1
  echo "launch list $w rc=$?"; tail -2 gpurun_out/r02_launches_$w.log
done
prof() {  # workload regex skip count
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s "$3" -c "$4" \
      -o "gpurun_out/r02_$1" -f python bench.py --workload "$1" --steps 12 --warmup 3 --no-cpu-baseline \
      > "gpurun_out/r02_ncu_$1.log" 2>&1
  echo "ncu $1 rc=$?"; tail -2 "gpurun_out/r02_ncu_$1.log"
  if [ -f "gpurun_out/r02_$1.ncu-rep" ]; then
    ncu -i "gpurun_out/r02_$1.ncu-rep" --page raw --csv > "gpurun_out/r02_ncu_$1_raw.csv" 2>/dev/null
    python tools/ncu_summary.py "gpurun_out/r02_$1.ncu-rep" > "gpurun_out/r02_ncu_$1.md" 2>&1
    rm -f "gpurun_out/r02_$1.ncu-rep"
  fi
}
prof svm1m "k_svm_chain|k_var_giant" 3 3
prof svm1m_rho2 "^k_svm_chain_w$" 1 1
prof pack5000 "k_collision_tiles_v3|k_var_row_pipe" 3 3
prof mpc100k "^k_mpc_block$" 1 1
du -sh gpurun_out
