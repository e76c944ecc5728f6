#!/bin/bash
# quick per-kernel bench of the listed workloads (under gpurun)
for w in "$@"; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "bench $w rc=$?"; tail -2 gpurun_out/bench_$w.err
  python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
d = json.load(open(f"gpurun_out/bench_{w}.json"))
print(f"{w}: {d['value']:.3e} EU/s  {d['ms_per_step']:.3f} ms/it  top={d['roofline']['kernel']} frac={d['roofline']['frac']:.3f}  e2e={d['e2e']['value']:.3e}")
print({k: (round(v['ms_avg'], 4), round(v['alg_bytes'] / v['ms_avg'] / 1e6) if v['ms_avg'] else 0) for k, v in d['kernels'].items()})
PY
done
