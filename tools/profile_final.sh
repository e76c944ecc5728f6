#!/bin/bash
# ncu --set full of each workload's top kernels + launch lists (1 GPU).
# Results: gpurun_out/final_<w>.ncu-rep, gpurun_out/launches_<w>.csv
set -u
mkdir -p gpurun_out
prof() {  # workload regex skip count
  ncu --set full --clock-control none --import-source on -k "regex:$2" -s "$3" -c "$4" \
      -o "gpurun_out/final_$1" -f python bench.py --workload "$1" --steps 3 --warmup 3 --no-cpu-baseline \
      > "gpurun_out/final_$1.log" 2>&1
  echo "ncu $1 rc=$?"
}
prof svm1m "k_svm_chain_unit|k_var_giant" 3 4
prof pack5000 "k_collision_tiles_v3|k_var_row_pipe|k_var_row_ring" 3 3
prof mpc100k "k_mpc_chain" 3 2
for w in svm1m pack5000 mpc100k; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$w.csv \
      python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "launch list $w rc=$?"
done
