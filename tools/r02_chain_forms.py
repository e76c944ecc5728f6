"""Per-form time of the fused SVM chain kernel at configs[1] (1M points x
32): unit weights, rho = 2 (power-of-two form), rho = 1.5 / alpha = 1.2
(refined reciprocals), and per-edge weights (every point's norm edge its
own rho and alpha via set_edge_params: the non-uniform weighted form).
Prints one JSON line per form with the chain kernel's CUDA-event time
(plan.profile_kernels) and its bandwidth against the copy peak.
Run under gpurun: python tools/r02_chain_forms.py [form ...]"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1603_02526_b200 as fg  # noqa: E402


def main():
    n = 1_000_000
    X, y = fg.gen_gaussian_arrays(n, 32, 4.0, seed=0)
    peak, kind = bench.measured_peak()
    want = sys.argv[1:] or ["unit", "pow2", "rcp", "per_edge"]
    for form, rho, alpha in [("unit", 1.0, 1.0), ("pow2", 2.0, 1.0), ("rcp", 1.5, 1.2),
                             ("per_edge", 1.0, 1.0)]:
        if form not in want:
            continue
        g = fg.build_svm(fg.SvmSpec.from_arrays(X, y, lam=1.0, rho=rho, alpha=alpha))
        if form == "per_edge":
            t0 = time.perf_counter()
            rng = np.random.default_rng(1)
            r = rng.uniform(0.5, 2.0, n)
            a = rng.uniform(0.8, 1.6, n)
            for i in range(n):                     # edge i: point i's norm edge
                g.set_edge_params(i, r[i], a[i])
            print(f"# per-edge weights set in {time.perf_counter() - t0:.1f} s", file=sys.stderr)
        st = fg.init_state(g)
        plan = fg.device_plan(g)
        plan.sync(g)
        plan.upload(st.z, st.u, st.n)
        plan.run(5)
        plan.upload(st.z, st.u, st.n)
        prof = plan.profile_kernels(22)
        ms, cnt = prof["chain_svm"]
        alg = bench.kernel_bytes(g, plan).get("chain_svm")
        line = {"form": form, "rho": rho, "alpha": alpha, "chain_form": plan.chain_form(),
                "forms": {k: v for k, v in plan.forms().items() if k.startswith("chain")},
                "chain_ms": ms / cnt, "launches": cnt}
        if alg:
            line["alg_bytes"] = alg
            line["GBps"] = alg / (ms / cnt) / 1e6
            line["frac"] = line["GBps"] / peak
            line["peak"] = [peak, kind]
        print(json.dumps(line), flush=True)
        del plan, g, st


if __name__ == "__main__":
    main()
