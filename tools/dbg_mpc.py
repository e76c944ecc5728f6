import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1603_02526_b200 as fg
w = sys.argv[1] if len(sys.argv) > 1 else "mpc100k"
g, st, _ = bench.build_instance(w)
plan = fg.device_plan(g)
plan.sync(g)
plan.upload(st.z, st.u, st.n)
plan.run(5)
for chunk in (2, 16, 64):
    for tol in (0.0, 1e-30):
        ts = []
        for r in range(6):
            res, _ = plan.run(64, primal_tol=tol, graph_chunk=chunk)
            ts.append(res.ms_total / 64)
        print(f"chunk {chunk} tol {tol}: " + " ".join(f"{t:.3f}" for t in ts))
