import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_02526_b200 as fg
from bench import ClockSampler
X, y = fg.gen_gaussian_arrays(1_000_000, 32, 4.0, seed=0)
g = fg.build_svm(fg.SvmSpec.from_arrays(X, y, lam=1.0))
st = fg.init_state(g)
plan = fg.device_plan(g)
plan.sync(g)
plan.upload(st.z, st.u, st.n)
plan.run(5)
for mode in ("none", "nvml5ms", "nvml20ms", "none"):
    ts = []
    for rep in range(12):
        if mode == "none":
            res, _ = plan.run(50, graph_chunk=16)
        else:
            with ClockSampler(0, 0.005 if mode == "nvml5ms" else 0.02):
                res, _ = plan.run(50, graph_chunk=16)
        ts.append(res.ms_total / 50)
    print(mode, " ".join(f"{t:.3f}" for t in ts))
