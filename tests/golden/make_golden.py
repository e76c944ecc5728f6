"""Generate golden vectors from the REFERENCE implementation.

Run in the container that has the reference mounted:

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py

Every array here comes from ``fgadmm`` itself (engine.run / iterate /
operators), never from this repo's engine or oracle.  Packing instances
are fully IEEE-portable (element-wise ops, 2-term einsum, pairwise sums),
so their results are pinned by SHA-256 of the raw float64 bytes; SVM and
MPC involve host-SIMD-dependent dots / LAPACK and are stored as arrays
(compared at 1e-9 relative).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import fgadmm  # noqa: E402
from fgadmm import problems as P  # noqa: E402
from support import two_quadratic_trace  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def copy_state(s):
    return fgadmm.AdmmState(*(getattr(s, k).copy() for k in "xmzun"), iteration=s.iteration)


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, sorted(arrays))


def run_ref(g, state, K, **kw):
    s = copy_state(state)
    _sol, rep = fgadmm.run(g, fgadmm.RunConfig(max_iterations=K, **kw), state=s)
    hist = np.array([[r[-2], r[-1]] for r in rep.history])
    return s, rep, hist


def packing():
    for n, iters in ((100, (1, 10, 1000)), (500, (10,))):
        spec = P.PackingSpec(n)
        g = P.build_packing(spec)
        st0 = P.packing_init(g, spec, seed=0)
        out = {"n": n, "init_sha": np.array([sha(getattr(st0, k)) for k in "xmzun"])}
        for K in iters:
            s, rep, hist = run_ref(g, st0, K)
            out[f"sha_{K}"] = np.array([sha(getattr(s, k)) for k in "xmzun"])
            out[f"z_{K}"] = s.z.copy()
            out[f"hist_{K}"] = hist
            if K <= 10 and n == 100:
                for k in "xmun":
                    out[f"{k}_{K}"] = getattr(s, k).copy()
        save(f"pack{n}_seed0.npz", **out)


def svm():
    pts = P.gen_gaussian_data(200, 32, 4.0, seed=0)
    g = P.build_svm(P.SvmSpec(pts, lam=1.0))
    out = {}
    for tag, st0 in (("zero", fgadmm.init_state(g)), ("seed1", fgadmm.init_state(g, seed=1))):
        s, rep, hist = run_ref(g, st0, 10)
        for k in "xmzun":
            out[f"{tag}_{k}_10"] = getattr(s, k).copy()
        out[f"{tag}_hist_10"] = hist
    X = np.stack([p.x for p in pts])
    out["X_sha"] = np.array(sha(X))
    save("svm200x32.npz", **out)


def mpc():
    spec = P.MpcSpec(10, fgadmm.LinearSystem(*P.pendulum_linearization()),
                     np.array([0.0, 0.0, 0.1, 0.0]))
    g = P.build_mpc(spec)
    st0 = fgadmm.init_state(g)
    out = {}
    s, rep, hist = run_ref(g, st0, 10)
    for k in "xmzun":
        out[f"{k}_10"] = getattr(s, k).copy()
    s, rep, hist = run_ref(g, st0, 100000, primal_tol=1e-9, dual_tol=1e-9)
    out["conv_iterations"] = np.array(rep.iterations)
    out["conv_z"] = s.z.copy()
    out["qp_solution"] = np.concatenate(P.mpc_qp_solution(spec))
    save("mpc_cartpole10.npz", **out)

    rng = np.random.default_rng(0)
    A = 0.05 * rng.standard_normal((16, 16))
    B = 0.1 * rng.standard_normal((16, 4))
    q0 = rng.standard_normal(16)
    spec = P.MpcSpec(50, fgadmm.LinearSystem(A, B), q0)
    g = P.build_mpc(spec)
    s, rep, hist = run_ref(g, fgadmm.init_state(g, seed=2), 10)
    out = {"A": A, "B": B, "q0": q0, "hist_10": hist}
    for k in "xmzun":
        out[f"{k}_10"] = getattr(s, k).copy()
    save("mpc16x4_T50.npz", **out)


def quadratic_trace():
    tr = two_quadratic_trace(3)
    out = {}
    for i, step in enumerate(tr):
        for k in "xmun":
            out[f"{k}_{i}"] = np.array([float(v) for v in step[k]])
        out[f"z_{i}"] = np.array([float(step["z"])])
    b = fgadmm.GraphBuilder()
    w = b.declare_variable(1)
    b.add_factor(fgadmm.Quadratic([[1.0]], [1.0]), [w])
    b.add_factor(fgadmm.Quadratic([[3.0]], [1.0]), [w])
    g = b.freeze()
    s = fgadmm.init_state(g)
    zp = s.z.copy()
    fgadmm.iterate(g, s)
    out["residuals_1"] = np.array(fgadmm.residuals(g, s, zp))
    save("two_quadratic.npz", **out)


def operators():
    """Random batches per kind evaluated by the reference batch_eval."""
    from fgadmm import operators as Op
    rng = np.random.default_rng(1234)
    B = 64
    out = {}

    def rho():
        return rng.uniform(0.1, 10.0, B)

    cases = {
        "collision": ({}, [rng.normal(size=(B, 2)), rng.uniform(0.1, 1, (B, 1)),
                           rng.normal(size=(B, 2)) * 0.3, rng.uniform(0.1, 1, (B, 1))],
                      [rho() for _ in range(4)]),
        "wall": ({"Q": np.tile([[0.6, 0.8]], (B, 1)), "V": rng.normal(size=(B, 2))},
                 [rng.normal(size=(B, 2)), rng.uniform(0, 1, (B, 1))], [rho(), rho()]),
        "radius": ({"kappa": np.full(B, 0.05)}, [rng.normal(size=(B, 1))],
                   [rng.uniform(0.1, 10, B)]),
        "svm_slack": ({"lam": rng.uniform(0, 2, B)}, [rng.normal(size=(B, 1))], [rho()]),
        "svm_norm": ({"scale": rng.uniform(0.01, 2, B)}, [rng.normal(size=(B, 32))], [rho()]),
        "svm_margin": ({"x": rng.normal(size=(B, 32)), "y": rng.choice([-1.0, 1.0], B)},
                       [rng.normal(size=(B, 32)), rng.normal(size=(B, 1)),
                        rng.normal(size=(B, 1))], [rho(), rho(), rho()]),
        "equality": ({}, [rng.normal(size=(B, 5)), rng.normal(size=(B, 5))], [rho(), rho()]),
        "mpc_cost": ({"diag": rng.uniform(0, 3, (B, 6))}, [rng.normal(size=(B, 6))], [rho()]),
        "mpc_init": ({"q0": rng.normal(size=(B, 4))}, [rng.normal(size=(B, 5))], [rho()]),
        "quadratic": ({"targets": [rng.normal(size=(B, 2)), rng.normal(size=(B, 1))],
                       "curvatures": [rng.uniform(0, 2, B), rng.uniform(0, 2, B)]},
                      [rng.normal(size=(B, 2)), rng.normal(size=(B, 1))], [rho(), rho()]),
    }
    A = 0.1 * rng.normal(size=(3, 3))
    Bm = 0.1 * rng.normal(size=(3, 2))
    sys_ = Op.LinearSystem(A, Bm)
    cases["mpc_dyn"] = ({"M": np.repeat(sys_.M[None], B, axis=0)},
                        [rng.normal(size=(B, 5)), rng.normal(size=(B, 5))], [rho(), rho()])
    out["mpc_dyn_A"], out["mpc_dyn_B"] = A, Bm
    for kind, (params, vals, rhos) in cases.items():
        cls = fgadmm.operator_class(kind)
        res = cls.batch_eval(params, vals, rhos)
        for j, v in enumerate(vals):
            out[f"{kind}_in{j}"] = v
            out[f"{kind}_rho{j}"] = rhos[j]
            out[f"{kind}_out{j}"] = res[j]
        for key, val in params.items():
            if key == "M":
                continue
            if isinstance(val, list):
                for j, a in enumerate(val):
                    out[f"{kind}_p_{key}{j}"] = a
            else:
                out[f"{kind}_p_{key}"] = val
    save("operators.npz", **out)


def converged():
    """Long runs of the reference for the convergence gates
    (``tests/test_gpu_convergence.py``; BASELINE.md "objective and
    feasibility at convergence", reference test_acceptance.py:157-192).

    Packing is bit-portable, so the device must reproduce the reference's
    state after 20,000 iterations exactly (SHA-256 of z), and with it the
    reference's objective and violation; the SVM N=12 case (C5) records
    the reference's converged solution and iteration count."""
    out = {}
    for n, K in ((100, 20000), (500, 20000)):
        spec = P.PackingSpec(n)
        g = P.build_packing(spec)
        st0 = P.packing_init(g, spec, seed=0)
        s, rep, hist = run_ref(g, st0, K, primal_tol=1e-8, dual_tol=1e-8,
                               record_every=1000)
        z = s.z.copy()
        out[f"pack{n}_iterations"] = np.array(rep.iterations)
        out[f"pack{n}_converged"] = np.array(rep.converged)
        out[f"pack{n}_sha"] = np.array([sha(getattr(s, k)) for k in "xmzun"])
        out[f"pack{n}_objective"] = np.array(g.objective_value(z))
        out[f"pack{n}_violation"] = np.array(g.constraint_violation(z))
        out[f"pack{n}_last_residuals"] = np.array(s.last_residuals)
        print(n, rep.iterations, rep.converged, out[f"pack{n}_objective"],
              out[f"pack{n}_violation"], flush=True)
    pts = P.gen_gaussian_data(12, 2, 4.0, seed=0)
    g = P.build_svm(P.SvmSpec(pts, lam=1.0))
    sol, rep = fgadmm.run(g, fgadmm.RunConfig(max_iterations=60000, primal_tol=1e-10,
                                              dual_tol=1e-10))
    out["svm12_iterations"] = np.array(rep.iterations)
    out["svm12_w"] = sol[0].copy()
    out["svm12_b"] = np.array(float(sol[12][0]))
    out["svm12_objective"] = np.array(P.svm_objective(pts, 1.0, sol[0], float(sol[12][0])))
    big = P.gen_gaussian_data(200, 2, 4.0, seed=0)
    g2 = P.build_svm(P.SvmSpec(big, lam=1.0))
    sol2, _ = fgadmm.run(g2, fgadmm.RunConfig(max_iterations=5000))
    out["svm200_w"] = sol2[0].copy()
    out["svm200_b"] = np.array(float(sol2[200][0]))
    out["svm200_accuracy"] = np.array(P.svm_accuracy(big, sol2[0], float(sol2[200][0])))
    save("converged.npz", **out)


def documents():
    """Graph documents written by the reference's ``serialize``
    (graph.py:265-286) and the reference's own 10-iteration results on the
    graphs it rebuilds from them (``deserialize``, graph.py:289-340): the
    device must run a document-driven graph to the same state.  Weights are
    varied per edge (set_edge_params) so the documents carry non-unit rho
    and alpha."""
    import gzip
    out = {}
    rng = np.random.default_rng(77)
    spec = P.PackingSpec(30)
    gp = P.build_packing(spec)
    for e in rng.choice(len(gp.edge_var), 40, replace=False):
        gp.set_edge_params(int(e), float(rng.uniform(0.5, 2.0)), float(rng.uniform(0.5, 1.5)))
    pts = P.gen_gaussian_data(60, 4, 4.0, seed=3)
    gs = P.build_svm(P.SvmSpec(pts, lam=0.7, rho=1.5, alpha=1.2))
    rng2 = np.random.default_rng(5)
    A = 0.05 * rng2.standard_normal((4, 4))
    B = 0.1 * rng2.standard_normal((4, 2))
    gm = P.build_mpc(P.MpcSpec(25, fgadmm.LinearSystem(A, B), rng2.standard_normal(4)))
    for tag, g0, seed in (("pack30", gp, 4), ("svm60x4", gs, 5), ("mpc4x2", gm, 6)):
        doc = fgadmm.serialize(g0)
        with gzip.open(os.path.join(HERE, f"doc_{tag}.json.gz"), "wt") as fh:
            fh.write(doc)
        g = fgadmm.deserialize(doc)
        assert fgadmm.serialize(g) == doc
        st0 = fgadmm.init_state(g, seed=seed)
        s, rep, hist = run_ref(g, st0, 10)
        for k in "xmzun":
            out[f"{tag}_{k}"] = getattr(s, k).copy()
        out[f"{tag}_sha"] = np.array([sha(getattr(s, k)) for k in "xmzun"])
        out[f"{tag}_hist"] = hist
        out[f"{tag}_doc_sha"] = np.array(hashlib.sha256(doc.encode()).hexdigest())
        out[f"{tag}_zmap"] = g.zmap.copy()
        out[f"{tag}_z_weights"] = g.z_weights.copy()
        out[f"{tag}_rho_flat"] = g.rho_flat.copy()
        out[f"{tag}_alpha_flat"] = g.alpha_flat.copy()
    save("documents.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["quadratic_trace", "operators", "packing", "svm", "mpc",
                             "documents", "converged"]
    for name in which:
        globals()[name]()
