#!/bin/bash
# run-to-run spread of the default bench line and the other workloads (same box, back to back)
set -u
mkdir -p gpurun_out
for rep in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/var_svm1m_$rep.json 2>/dev/null
  for w in pack5000 mpc100k; do
    timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/var_${w}_$rep.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob
for w in ("svm1m", "pack5000", "mpc100k"):
    rows = []
    for f in sorted(glob.glob(f"gpurun_out/var_{w}_*.json")):
        d = json.load(open(f))
        rows.append((d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"]))
    print(w, rows)
PY
