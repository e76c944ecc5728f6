mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_var_giant_chunks" -s 2 -c 1 -o gpurun_out/g_chunks -f python bench.py --workload svm1m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g_chunks.log 2>&1
ncu -i gpurun_out/g_chunks.ncu-rep --page details --csv > gpurun_out/g_chunks_details.csv 2>/dev/null
ncu -i gpurun_out/g_chunks.ncu-rep --page source --csv --print-source sass > gpurun_out/g_chunks_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/g_chunks.ncu-rep > gpurun_out/g_chunks.md 2>&1
rm -f gpurun_out/g_chunks.ncu-rep
cat gpurun_out/g_chunks.md
