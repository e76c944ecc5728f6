import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1603_02526_b200 as fg
import bench
import scipy.sparse as sp, scipy.sparse.linalg as spla

def mpc_kkt_sparse(A, B, q0, T):
    d, k = B.shape; w = d + k; nvar = (T + 1) * w
    F = np.eye(d) + A
    rows, cols, vals = [], [], []
    def add(r0, c0, M):
        M = np.asarray(M); ii, jj = np.nonzero(M)
        rows.extend(r0 + ii); cols.extend(c0 + jj); vals.extend(M[ii, jj])
    add(0, 0, np.eye(d))
    for t in range(T):
        r = d * (t + 1)
        add(r, t * w, -F); add(r, t * w + d, -B); add(r, (t + 1) * w, np.eye(d))
    Aeq = sp.csr_matrix((vals, (rows, cols)), shape=(d * (T + 1), nvar))
    beq = np.zeros(d * (T + 1)); beq[:d] = q0
    K = sp.bmat([[sp.identity(nvar), Aeq.T], [Aeq, None]], format="csc")
    sol = spla.spsolve(K, np.concatenate([np.zeros(nvar), beq]))
    return sol[:nvar]

for T in (1000, 100000):
    g, st, info = bench.build_instance("mpc100k", T / 100000)
    rng = np.random.default_rng(0)
    A = 0.05 * rng.standard_normal((16, 16)); B = 0.1 * rng.standard_normal((16, 4)); q0 = rng.standard_normal(16)
    t = time.time(); ref = mpc_kkt_sparse(A, B, q0, T); tk = time.time() - t
    for tol in (1e-7, 1e-9):
        s = fg.init_state(g)
        sol, rep = fg.run(g, fg.RunConfig(max_iterations=300000, primal_tol=tol, dual_tol=tol, record_every=100000), state=s)
        z = sol.concatenated()
        print("mpc", T, tol, rep.iterations, rep.converged, float(np.max(np.abs(z - ref))), "kkt s", round(tk, 1), "dev s", rep.device_seconds, flush=True)

for n in (2000,):
    pts = fg.gen_gaussian_data(n, 32, 4.0, seed=0)
    g = fg.build_svm(fg.SvmSpec(pts, lam=1.0))
    t = time.time(); qp = fg.svm_qp_solution(pts, 1.0); tq = time.time() - t
    for tol in (1e-7, 1e-9):
        sol, rep = fg.run(g, fg.RunConfig(max_iterations=300000, primal_tol=tol, dual_tol=tol, record_every=100000))
        w, b = sol[0], float(sol[n][0])
        obj = fg.svm_objective(pts, 1.0, w, b)
        print("svm", n, tol, rep.iterations, rep.converged, obj, qp["objective"], abs(obj - qp["objective"]) / abs(qp["objective"]), "qp s", round(tq, 1), flush=True)

for n in (500, 5000):
    g, st, info = bench.build_instance("pack5000", n / 5000) if n == 5000 else (None, None, None)
    if g is None:
        spec = fg.PackingSpec(n); g = fg.build_packing(spec); st = fg.packing_init(g, spec, seed=0)
    for K in (20000, 100000):
        s = fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun"))
        sol, rep = fg.run(g, fg.RunConfig(max_iterations=K, primal_tol=1e-8, dual_tol=1e-8, record_every=K), state=s)
        z = sol.concatenated()
        print("pack", n, K, rep.iterations, rep.converged, fg.engine.objective_value(g, z), fg.engine.constraint_violation(g, z), rep.history[-1][-2:], rep.device_seconds, flush=True)
