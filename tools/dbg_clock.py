"""Graph-path run-to-run variance with the GPU kept busy vs idle gaps."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1603_02526_b200 as fg
w = sys.argv[1]
g, st, _ = bench.build_instance(w)
plan = fg.device_plan(g)
plan.sync(g)
plan.upload(st.z, st.u, st.n)
plan.run(6)
for label, gap in (("back-to-back", 0.0), ("50ms idle gap", 0.05)):
    ts = []
    for r in range(8):
        if gap:
            time.sleep(gap)
            plan.run(6)          # warm-up right before, like bench.py
        res, _ = plan.run(50)
        ts.append(res.ms_total / 50)
    print(w, label, " ".join(f"{t:.3f}" for t in ts))
