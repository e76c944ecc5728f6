"""Randomized irregular graphs on the device: variables of mixed dims,
quadratic factors of 1-3 slots on random variables and equality factors
between random same-dim variables, interleaved in creation order (so most
groups fall back to the per-slot index tables instead of affine runs),
hub variables whose degree crosses the small / large / giant class
boundaries, random per-edge rho and alpha, random initial state.  Every
kind involved is an exact closed form, so the device state must equal the
oracle's bit for bit after several iterations (the oracle is pinned to the
reference, tests/test_oracle.py)."""

import numpy as np
import pytest

import paper_1603_02526_b200 as fg
from oracle import fgadmm_oracle as O

pytestmark = pytest.mark.gpu


def random_graph(seed, nv=60, nf=400, hub_degrees=(40, 300)):
    rng = np.random.default_rng(seed)
    dims = rng.choice([1, 2, 3, 5], size=nv, p=[0.3, 0.3, 0.2, 0.2])
    b = fg.GraphBuilder()
    ids = [b.declare_variable(int(d)) for d in dims]
    by_dim = {d: [v for v in ids if dims[v] == d] for d in set(dims.tolist())}

    def quad(vs):
        t = [rng.standard_normal(int(dims[v])) for v in vs]
        c = rng.uniform(0.0, 3.0, size=len(vs))
        b.add_factor(fg.Quadratic(t, c), vs, rho=float(rng.choice([1.0, 0.5, 2.0, 1.3])),
                     alpha=float(rng.choice([1.0, 1.5, 0.8])))

    for _ in range(nf):
        if rng.random() < 0.7:
            k = int(rng.integers(1, 4))
            quad([int(v) for v in rng.choice(nv, size=k, replace=False)])
        else:
            d = int(rng.choice([d for d, vs in by_dim.items() if len(vs) >= 2]))
            a, c = rng.choice(by_dim[d], size=2, replace=False)
            b.add_factor(fg.Equality(d), [int(a), int(c)], rho=float(rng.choice([1.0, 0.7, 2.0])))
    # hubs: one variable per requested degree gets that many unary quadratics
    for deg in hub_degrees:
        h = int(rng.integers(0, nv))
        for _ in range(deg):
            quad([h])
    g = b.freeze()
    # a sample of edges re-weighted after freezing (set_edge_params)
    for e in rng.choice(len(g.edge_var), size=min(50, len(g.edge_var)), replace=False):
        g.set_edge_params(int(e), float(rng.uniform(0.2, 3.0)), float(rng.uniform(0.5, 1.8)))
    return g


@pytest.mark.parametrize("seed,hubs", [(1, (40, 300)), (2, (9, 33)), (3, (8200, 50)),
                                       (4, (5,)), (5, (1000, 2000, 9000)), (6, (64, 129))])
def test_random_irregular_graph_bitwise_vs_oracle(gpu, seed, hubs):
    g = random_graph(seed, hub_degrees=hubs)
    st = fg.init_state(g, seed=seed)
    s = fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun"))
    _sol, rep = fg.run(g, fg.RunConfig(max_iterations=7), state=s)
    ref, hist, _ = O.run(g, 7, st)
    assert rep.iterations == 7
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(s, k), getattr(ref, k), err_msg=k)
    dev = np.array([h[-2:] for h in rep.history])
    np.testing.assert_allclose(dev, np.array(hist), rtol=1e-12)


@pytest.mark.parametrize("seed", [7, 8])
def test_random_irregular_graph_tolerance_stop_and_resume(gpu, seed):
    """The same graphs under a tolerance stop, then resumed from the
    returned state: the device stops at the oracle's iteration with the
    oracle's state."""
    g = random_graph(seed, nv=40, nf=200, hub_degrees=(50,))
    st = fg.init_state(g, seed=seed)
    s = fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun"))
    _sol, rep = fg.run(g, fg.RunConfig(max_iterations=400, primal_tol=1e-3, dual_tol=1e-3),
                       state=s)
    ref, hist, conv = O.run(g, 400, st, primal_tol=1e-3, dual_tol=1e-3)
    assert conv                            # stops near iteration 180
    assert rep.converged == conv and rep.iterations == len(hist)
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(s, k), getattr(ref, k), err_msg=k)
    _sol, rep2 = fg.run(g, fg.RunConfig(max_iterations=5), state=s)
    ref2, _h, _ = O.run(g, 5, ref)
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(s, k), getattr(ref2, k), err_msg=k)


def random_mixed_graph(seed, nd=30, npair=150):
    """Packing-kind factors in an irregular arrangement (random disk pairs,
    not the all-pairs triangle: the generic collision kernel and per-slot
    tables), random walls and radii, plus SVM norm / slack and MPC cost /
    init factors on their own variables, interleaved with equalities."""
    rng = np.random.default_rng(seed)
    b = fg.GraphBuilder()
    c = [b.declare_variable(2) for _ in range(nd)]
    r = [b.declare_variable(1) for _ in range(nd)]
    w = [b.declare_variable(4) for _ in range(10)]
    xi = [b.declare_variable(1) for _ in range(10)]
    nodes = [b.declare_variable(5) for _ in range(8)]
    planes = [fg.HalfPlane([0.0, 1.0], [0.0, 0.0]), fg.HalfPlane([1.0, -1.0], [0.5, 0.0])]
    for _ in range(npair):
        i, j = (int(v) for v in rng.choice(nd, size=2, replace=False))
        b.add_factor(fg.Collision(), [c[i], r[i], c[j], r[j]], rho=float(rng.choice([1.0, 2.0, 0.6])))
        u = rng.random()
        if u < 0.2:
            k = int(rng.integers(nd))
            b.add_factor(fg.Wall(planes[int(rng.integers(2))]), [c[k], r[k]])
        elif u < 0.3:
            k = int(rng.integers(nd))
            b.add_factor(fg.Radius(0.5), [r[k]], rho=float(rng.choice([5.0, 3.0])))
        elif u < 0.4:
            k = int(rng.integers(10))
            b.add_factor(fg.SvmNorm(0.01, 4), [w[k]], rho=float(rng.choice([1.0, 1.5])))
        elif u < 0.5:
            k = int(rng.integers(10))
            b.add_factor(fg.SvmSlack(0.7), [xi[k]])
        elif u < 0.6:
            k = int(rng.integers(8))
            b.add_factor(fg.MpcCost(rng.uniform(0.5, 2.0, 3), rng.uniform(0.5, 2.0, 2)), [nodes[k]])
        elif u < 0.7:
            a2, b2 = (int(v) for v in rng.choice(10, size=2, replace=False))
            b.add_factor(fg.Equality(4), [w[a2], w[b2]], alpha=1.3)
    b.add_factor(fg.MpcInit(rng.standard_normal(3), 2), [nodes[0]])
    for v in w + xi + nodes:                       # every variable has an edge
        b.add_factor(fg.Quadratic([np.zeros(b._dims[v])], [1.0]), [v])
    return b.freeze()


@pytest.mark.parametrize("seed", [11, 12, 13, 14])
def test_random_mixed_kinds_bitwise_vs_oracle(gpu, seed):
    g = random_mixed_graph(seed)
    st = fg.init_state(g, seed=seed)
    s = fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun"))
    fg.run(g, fg.RunConfig(max_iterations=9), state=s)
    ref, _h, _ = O.run(g, 9, st)
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(s, k), getattr(ref, k), err_msg=k)
