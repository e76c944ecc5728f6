import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1603_02526_b200 as fg
from bench import ClockSampler
X, y = fg.gen_gaussian_arrays(1_000_000, 32, 4.0, seed=0)
g = fg.build_svm(fg.SvmSpec.from_arrays(X, y, lam=1.0))
st = fg.init_state(g)
plan = fg.device_plan(g)
plan.sync(g)
plan.upload(st.z, st.u, st.n)
plan.run(5)
for rep in range(3):
    for chunk in (2, 16, 64):
        for K in (20, 50, 200):
            with ClockSampler(0, 0.002) as clk:
                res, _ = plan.run(K, graph_chunk=chunk)
            c = clk.summary()
            print(f"rep {rep} chunk {chunk} K {K}: {res.ms_total / K:.4f} ms/it  sm {c['sm_mhz']} {c['reasons']}")
res, _ = plan.run(50, timing=True)
print(f"timing path: {res.ms_total / 50:.4f} ms/it edge {res.ms_edge_pass/50:.4f} var {res.ms_var_pass/50:.4f} red {res.ms_reduce/50:.4f}")
