"""Repeated device timing of a workload's fused loop (distribution, not one
sample): python tools/rep_timing.py <workload> [reps] [K]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1603_02526_b200 as fg
w = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
K = int(sys.argv[3]) if len(sys.argv) > 3 else 50
g, st, _ = bench.build_instance(w)
plan = fg.device_plan(g)
plan.sync(g)
plan.upload(st.z, st.u, st.n)
plan.run(5)
ts = []
for r in range(reps):
    res, _ = plan.run(K)
    ts.append(res.ms_total / K)
res, _ = plan.run(K, timing=True)
prof = plan.profile_kernels(10)
print(w, "ms/it min %.4f med %.4f max %.4f" % (min(ts), float(np.median(ts)), max(ts)),
      "| timing-path %.4f" % (res.ms_total / K), "| kernel sum %.4f" %
      sum(v[0] / v[1] for v in prof.values()))
print("  ", " ".join(f"{t:.3f}" for t in ts))
print("  ", {k: round(v[0] / v[1], 4) for k, v in prof.items()})
