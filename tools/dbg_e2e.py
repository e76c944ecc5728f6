"""Host-side breakdown of one public run() call on a bench workload."""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
import bench
import paper_1603_02526_b200 as fg
from paper_1603_02526_b200 import engine

name = sys.argv[1] if len(sys.argv) > 1 else "svm1m"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
g, st, info = bench.build_instance(name)
s = fg.pinned_state(g, st)
cfg = engine.RunConfig(max_iterations=K)
engine.run(g, cfg, state=fg.pinned_state(g, st))
plan = engine.device_plan(g)
for rep in range(3):
    T = {}
    t = time.perf_counter()
    plan.host_checks(g); T["host_checks"] = time.perf_counter() - t; t = time.perf_counter()
    plan.sync(g); T["sync"] = time.perf_counter() - t; t = time.perf_counter()
    plan.upload(s.z, s.u, s.n); T["upload"] = time.perf_counter() - t; t = time.perf_counter()
    res, hist = plan.run(K); T["run"] = time.perf_counter() - t; t = time.perf_counter()
    T["dev_ms"] = res.ms_total / 1e3
    plan.download(x=s.x, m=s.m, z=s.z, u=s.u, n=s.n); T["download"] = time.perf_counter() - t
    t = time.perf_counter()
    engine._nonfinite_message(g, s.n, "n", K); T["nscan"] = time.perf_counter() - t
    t = time.perf_counter()
    engine.run(g, cfg, state=s); T["run()"] = time.perf_counter() - t
    print(name, " ".join(f"{k} {v*1e3:.1f}ms" for k, v in T.items()), flush=True)
