"""CPU ORACLE — test infrastructure only.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and
only as the checker or the timed CPU baseline; the product path
(``paper_1603_02526_b200``) never calls it.

A NumPy restatement of the reference's five-phase iteration
(``/root/reference/pkg/src/fgadmm/engine.py``) and closed-form operators
(``.../operators.py``) on the flat edge-ordered arrays of a frozen graph.
It issues the same NumPy operations in the same order as the reference
(take / multiply / add.reduceat / divide / einsum / linalg.solve /
linalg.norm), so on one host it is bit-identical to the reference; that
is pinned by ``tests/test_oracle.py`` against the reference itself (when
``/root/reference`` is present) and against the committed golden vectors
in ``tests/golden/`` (generated from the reference by
``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import time

import numpy as np


# ---------------------------------------------------------------------------
# closed-form proximal maps; values/rhos are per-slot (B, d) / (B,) arrays

def _prox_quadratic(p, vals, rhos):                     # operators.py:131-135
    return [(C[:, None] * T + R[:, None] * N) / (C + R)[:, None]
            for T, C, N, R in zip(p["targets"], p["curvatures"], vals, rhos)]


def _prox_collision(p, vals, rhos):                     # operators.py:166-191
    a_c, a_r, b_c, b_r = vals
    w_ac, w_ar, w_bc, w_br = rhos
    delta = a_c - b_c
    length = np.sqrt(np.einsum("bi,bi->b", delta, delta))
    unit = delta / np.where(length > 0.0, length, 1.0)[:, None]
    unit[length == 0.0] = (-1.0, 0.0)
    overlap = np.maximum(a_r[:, 0] + b_r[:, 0] - length, 0.0)
    mult = overlap / (1.0 / w_ac + 1.0 / w_bc + 1.0 / w_ar + 1.0 / w_br)
    return [a_c + (mult / w_ac)[:, None] * unit,
            a_r - (mult / w_ar)[:, None],
            b_c - (mult / w_bc)[:, None] * unit,
            b_r - (mult / w_br)[:, None]]


def _prox_wall(p, vals, rhos):                          # operators.py:226-234
    c, r = vals
    wc, wr = rhos
    normal, anchor = p["Q"], p["V"]
    gap = np.einsum("bi,bi->b", normal, c - anchor) - r[:, 0]
    mult = np.maximum(-gap, 0.0) / (1.0 / wc + 1.0 / wr)
    return [c + (mult / wc)[:, None] * normal, r - (mult / wr)[:, None]]


def _prox_radius(p, vals, rhos):                        # operators.py:272-277
    (N,), (R,) = vals, rhos
    if np.any(R <= p["kappa"]):
        raise ValueError("radius prox requires rho > kappa")
    return [R[:, None] * N / (R - p["kappa"])[:, None]]


def _prox_mpc_cost(p, vals, rhos):                      # operators.py:312-314
    (N,), (R,) = vals, rhos
    return [R[:, None] * N / (p["diag"] + R[:, None])]


def _prox_mpc_init(p, vals, rhos):                      # operators.py:349-354
    out = vals[0].copy()
    q0 = np.asarray(p["q0"])
    out[:, :q0.shape[1]] = q0
    return [out]


def _stacked_M(p):
    if "M" in p:
        return np.asarray(p["M"])
    Ms = np.stack([np.asarray(s.M, dtype=float) for s in p["systems"]])
    return Ms[np.asarray(p["index"], dtype=np.int64)]


def _prox_mpc_dyn(p, vals, rhos):                       # operators.py:86-96, 390-404
    N0, N1 = vals
    R0, R1 = rhos
    M = _stacked_M(p)
    d = M.shape[1]
    k0 = N0.shape[1]
    nv = np.concatenate([N0, N1[:, :d]], axis=1)
    w = np.concatenate([np.repeat(R0[:, None], k0, axis=1),
                        np.repeat(R1[:, None], d, axis=1)], axis=1)
    winv = 1.0 / w
    Mn = np.einsum("bij,bj->bi", M, nv)
    S = np.einsum("bij,bj,bkj->bik", M, winv, M)
    lam = np.linalg.solve(S, Mn[..., None])[..., 0]
    v = nv - winv * np.einsum("bij,bi->bj", M, lam)
    tail = N1.copy()
    tail[:, :d] = v[:, k0:]
    return [v[:, :k0], tail]


def _prox_svm_slack(p, vals, rhos):                     # operators.py:439-441
    (N,), (R,) = vals, rhos
    return [np.maximum(N - (p["lam"] / R)[:, None], 0.0)]


def _prox_svm_norm(p, vals, rhos):                      # operators.py:477-479
    (N,), (R,) = vals, rhos
    return [(R / (R + p["scale"]))[:, None] * N]


def _prox_svm_margin(p, vals, rhos):                    # operators.py:515-525
    w, b, xi = vals
    rw, rb, rx = rhos
    X, Y = p["x"], p["y"]
    short = 1.0 - xi[:, 0] - Y * (np.einsum("bi,bi->b", w, X) + b[:, 0])
    mult = np.maximum(short, 0.0) / (np.einsum("bi,bi->b", X, X) / rw + 1.0 / rb + 1.0 / rx)
    return [w + (mult / rw * Y)[:, None] * X,
            b + (mult / rb * Y)[:, None],
            xi + (mult / rx)[:, None]]


def _prox_equality(p, vals, rhos):                      # operators.py:560-564
    N1, N2 = vals
    R1, R2 = rhos
    mean = (R1[:, None] * N1 + R2[:, None] * N2) / (R1 + R2)[:, None]
    return [mean, mean.copy()]


def _prox_nan_test(p, vals, rhos):
    out = vals[0].copy()
    for i, mode in enumerate(p["mode"]):
        if mode == "raise":
            raise FloatingPointError("synthetic failure")
        if mode == "nan":
            out[i] = np.nan
    return [out]


PROX = {
    "quadratic": _prox_quadratic, "collision": _prox_collision, "wall": _prox_wall,
    "radius": _prox_radius, "mpc_cost": _prox_mpc_cost, "mpc_init": _prox_mpc_init,
    "mpc_dyn": _prox_mpc_dyn, "svm_slack": _prox_svm_slack, "svm_norm": _prox_svm_norm,
    "svm_margin": _prox_svm_margin, "equality": _prox_equality, "nan_test": _prox_nan_test,
}


def prox_batch(kind, params, values, rhos):
    """Closed-form prox of one (kind) batch, restated from operators.py."""
    return PROX[kind](params, [np.asarray(v, dtype=float) for v in values],
                      [np.asarray(r, dtype=float) for r in rhos])


# ---------------------------------------------------------------------------
# the five phases on flat arrays (engine.py:113-309, single lane)

class Oracle:
    """Per-graph tables of the reference engine (_GraphOps, engine.py:166-189)."""

    def __init__(self, graph):
        self.g = graph
        self.groups = []
        for cls, dims, f0, _vars, params in self._blocks(graph):
            self.groups.append((cls.kind, dims, self._slot_index(graph, dims, f0, len(_vars)),
                                params))
        self.z_order = np.argsort(graph.zmap, kind="stable")
        self.z_ptr = np.searchsorted(graph.zmap[self.z_order],
                                     np.arange(graph.z_dim + 1, dtype=np.int64), side="left")

    @staticmethod
    def _blocks(graph):
        if hasattr(graph, "blocks"):
            return graph.blocks
        # a reference-package graph: one block per factor run of one kind
        out, run = [], []
        for f in graph.factors:
            key = (type(f.operator), tuple(f.operator.slot_dims()))
            if run and run[0][0] != key:
                out.append(Oracle._pack(run))
                run = []
            run.append((key, f))
        if run:
            out.append(Oracle._pack(run))
        return out

    @staticmethod
    def _pack(run):
        (cls, dims), f0 = run[0][0], run[0][1].id
        ops = [f.operator for _k, f in run]
        return cls, dims, f0, np.zeros((len(ops), len(dims))), cls.stack_params(ops)

    @staticmethod
    def _slot_index(graph, dims, f0, count):
        # edges of factor f0+i are consecutive; slot j -> edge e0+j
        if hasattr(graph, "factor_first_edges"):
            e0 = graph._factor_edge0[f0:f0 + count]
        else:
            e0 = np.array([graph.factors[f0 + i].edge_range[0] for i in range(count)],
                          dtype=np.int64)
        idx = []
        for j, d in enumerate(dims):
            starts = graph.edge_offsets[e0 + j]
            idx.append((starts[:, None] + np.arange(d, dtype=np.int64), e0 + j))
        return idx

    # phase x (engine.py:257-261, 140-151)
    def phase_x(self, s):
        for kind, _dims, idx, params in self.groups:
            vals = [s.n[i] for i, _e in idx]
            rhos = [self.g.edge_rho[e] for _i, e in idx]
            out = prox_batch(kind, params, vals, rhos)
            for (i, _e), o in zip(idx, out):
                s.x[i] = o

    def phase_m(self, s):                               # engine.py:263-265
        np.add(s.x, s.u, out=s.m)

    def phase_z(self, s):                               # engine.py:267-280
        vals = np.take(s.m, self.z_order) * np.take(self.g.rho_flat, self.z_order)
        sums = np.add.reduceat(vals, self.z_ptr[:-1])
        np.divide(sums, self.g.z_weights, out=s.z)

    def phase_u(self, s):                               # engine.py:282-290
        step = (s.x - np.take(s.z, self.g.zmap)) * self.g.alpha_flat
        np.add(s.u, step, out=s.u)

    def phase_n(self, s):                               # engine.py:292-298
        np.subtract(np.take(s.z, self.g.zmap), s.u, out=s.n)

    def iterate(self, s):
        for name in ("x", "m", "z", "u", "n"):
            getattr(self, "phase_" + name)(s)

    def residuals(self, s, z_prev):                     # engine.py:398-406
        scale = 1.0 / np.sqrt(self.g.total_edge_payload)
        primal = np.linalg.norm(s.x - s.z[self.g.zmap]) * scale
        dual = np.linalg.norm(self.g.rho_flat * (s.z - z_prev)[self.g.zmap]) * scale
        return float(primal), float(dual)


class State:
    """Plain holder of the five arrays (like AdmmState)."""

    def __init__(self, x, m, z, u, n):
        self.x, self.m, self.z, self.u, self.n = x, m, z, u, n

    @classmethod
    def copy_of(cls, st):
        return cls(*(np.array(getattr(st, k), dtype=float, copy=True) for k in "xmzun"))


def run(graph, iterations, state, primal_tol=0.0, dual_tol=0.0, oracle=None):
    """The reference run loop (engine.py:483-516), residuals every
    iteration; returns (state, history [(primal, dual)], converged)."""
    o = oracle or Oracle(graph)
    s = State.copy_of(state)
    hist = []
    converged = False
    for _it in range(iterations):
        z_prev = s.z.copy()
        o.iterate(s)
        pr, du = o.residuals(s, z_prev)
        hist.append((pr, du))
        checks = []
        if primal_tol > 0.0:
            checks.append(pr <= primal_tol)
        if dual_tol > 0.0:
            checks.append(du <= dual_tol)
        if checks and all(checks):
            converged = True
            break
    return s, hist, converged


def time_iterations(graph, state, iterations, oracle=None):
    """Seconds per iteration of the phase loop (CPU baseline timing)."""
    o = oracle or Oracle(graph)
    s = State.copy_of(state)
    t0 = time.perf_counter()
    for _ in range(iterations):
        o.iterate(s)
    return (time.perf_counter() - t0) / iterations, s


# ---------------------------------------------------------------------------
# partitioned restatement (checker for the multi-GPU protocol)

def run_partitioned(lg, iterations, state, allgather):
    """The five phases on one rank's LocalGraph ``lg``: non-cut variables
    as in ``Oracle``; cut variables from the rank-order sum of all-gathered
    local partials.  ``allgather(vec) -> [vec_rank0, vec_rank1, ...]``.
    Returns (local state, [(primal, dual)])."""
    from paper_1603_02526_b200.partition import combine_partials, local_partial_sums
    o = Oracle(lg)
    s = State.copy_of(state)
    cut = lg.cut_index >= 0
    P_global = None
    hist = []
    for _ in range(iterations):
        z_prev = s.z.copy()
        o.phase_x(s)
        o.phase_m(s)
        o.phase_z(s)
        if lg.ncut:
            tot = combine_partials(allgather(local_partial_sums(lg, s.m)))
            s.z[cut] = tot[lg.cut_index[cut]] / lg.z_weights[cut]
        o.phase_u(s)
        o.phase_n(s)
        d1 = s.x - s.z[lg.zmap]
        d2 = lg.rho_flat * (s.z - z_prev)[lg.zmap]
        parts = allgather(np.array([float(d1 @ d1), float(d2 @ d2),
                                    float(lg.total_edge_payload)]))
        tot = combine_partials(parts)
        P_global = tot[2]
        scale = 1.0 / np.sqrt(P_global)
        hist.append((float(np.sqrt(tot[0]) * scale), float(np.sqrt(tot[1]) * scale)))
    return s, hist
