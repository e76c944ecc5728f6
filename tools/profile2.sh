#!/bin/bash
# ncu --set full captures of the top kernels of pack5000 and svm1m + launch lists
set -u
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:k_collision_tiles_reg|k_var_large_vec" -s 6 -c 3 \
    -o gpurun_out/full_pack5000 -f python bench.py --workload pack5000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/full_pack5000.log 2>&1
echo "ncu pack rc=$?"
ncu --set full --clock-control none --import-source on -k "regex:k_var_small_run|k_svm_margin|k_elementwise|k_var_giant" -s 12 -c 8 \
    -o gpurun_out/full_svm1m -f python bench.py --workload svm1m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/full_svm1m.log 2>&1
echo "ncu svm rc=$?"
for w in svm1m pack5000 mpc100k; do
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$w.csv \
    python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "launch list $w rc=$?"
done
