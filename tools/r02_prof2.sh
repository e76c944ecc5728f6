#!/bin/bash
# ncu --set full of the weighted SVM chain and the blocked MPC chain, with
# the raw and source pages exported on the box (gpurun_out/r02_p2_*)
set -u
mkdir -p gpurun_out
prof() {  # tag workload regex skip count steps
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$3" -s "$4" -c "$5" \
      -o "gpurun_out/r02_p2_$1" -f python bench.py --workload "$2" --steps "$6" --warmup 3 --no-cpu-baseline \
      > "gpurun_out/r02_p2_$1.log" 2>&1
  echo "ncu $1 rc=$?"; tail -2 "gpurun_out/r02_p2_$1.log"
  if [ -f "gpurun_out/r02_p2_$1.ncu-rep" ]; then
    ncu -i "gpurun_out/r02_p2_$1.ncu-rep" --page raw --csv > "gpurun_out/r02_p2_$1_raw.csv" 2>/dev/null
    ncu -i "gpurun_out/r02_p2_$1.ncu-rep" --page source --csv --print-source sass > "gpurun_out/r02_p2_$1_sass.csv" 2>/dev/null
    ncu -i "gpurun_out/r02_p2_$1.ncu-rep" --page details --csv > "gpurun_out/r02_p2_$1_details.csv" 2>/dev/null
    python tools/ncu_summary.py "gpurun_out/r02_p2_$1.ncu-rep" > "gpurun_out/r02_p2_$1.md" 2>&1
    rm -f "gpurun_out/r02_p2_$1.ncu-rep"
  fi
}
prof chainw svm1m_rho2 "k_svm_chain_w" 1 1 3
prof mpcblock mpc100k "k_mpc_block" 1 1 12
prof rowd1 pack5000 "k_var_row_pipe" 1 2 3
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_mpc100k.csv \
    python bench.py --workload mpc100k --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/r02_launches_mpc100k.log 2>&1
echo "launch list mpc rc=$?"
timeout 600 python -m pytest tests/test_gpu_nccl.py -q -p no:cacheprovider 2>&1 | tail -3
du -sh gpurun_out
