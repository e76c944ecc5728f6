"""Engine API semantics on the device, mirroring the reference engine tests
(``tests/test_engine.py``): config validation, state checks, tolerance
stop, history stride, resume, fault messages, operator known answers."""

import numpy as np
import pytest

from conftest import golden
import paper_1603_02526_b200 as fg
from oracle import fgadmm_oracle as O

pytestmark = pytest.mark.gpu


def two_quadratic_graph():
    b = fg.GraphBuilder()
    w = b.declare_variable(1)
    b.add_factor(fg.Quadratic([[1.0]], [1.0]), [w])
    b.add_factor(fg.Quadratic([[3.0]], [1.0]), [w])
    return b.freeze()


def test_run_config_validation(gpu):
    g = two_quadratic_graph()
    for cfg in (fg.RunConfig(max_iterations=0), fg.RunConfig(max_iterations=1, workers=0),
                fg.RunConfig(max_iterations=1, record_every=0)):
        with pytest.raises(ValueError):
            fg.run(g, cfg)


def test_run_rejects_mismatched_state(gpu):
    g = two_quadratic_graph()
    s = fg.init_state(fg.build_packing(fg.PackingSpec(2)))
    with pytest.raises(ValueError):
        fg.run(g, fg.RunConfig(max_iterations=1), state=s)


def test_consensus_and_tolerance_stop(gpu):
    g = two_quadratic_graph()
    sol, rep = fg.run(g, fg.RunConfig(max_iterations=200))
    assert abs(sol[0][0] - 2.0) <= 1e-6 and rep.iterations == 200 and not rep.converged
    sol, rep = fg.run(g, fg.RunConfig(max_iterations=500, primal_tol=1e-9, dual_tol=1e-9))
    assert rep.converged and rep.iterations < 200
    assert abs(sol[0][0] - 2.0) <= 1e-6
    # the converged iteration equals the oracle's
    st = fg.init_state(g)
    _s, hist, conv = O.run(g, 500, st, 1e-9, 1e-9)
    assert conv and len(hist) == rep.iterations


def test_history_stride_and_report(gpu):
    g = two_quadratic_graph()
    _sol, rep = fg.run(g, fg.RunConfig(max_iterations=10, record_every=3))
    lines = rep.metrics_csv().strip().split("\n")
    assert lines[0] == fg.METRICS_HEADER
    assert [int(r.split(",")[0]) for r in lines[1:]] == [3, 6, 9, 10]
    assert rep.total_seconds >= sum(rep.phase_seconds.values())
    assert set(rep.phase_seconds) == set(fg.PHASES)
    assert rep.time_per_iteration() > 0.0


def test_run_continues_from_prior_state(gpu):
    g = two_quadratic_graph()
    s = fg.init_state(g)
    fg.run(g, fg.RunConfig(max_iterations=3), state=s)
    assert s.iteration == 3
    fg.run(g, fg.RunConfig(max_iterations=2), state=s)
    assert s.iteration == 5
    fresh, _ = fg.run(g, fg.RunConfig(max_iterations=5))
    np.testing.assert_array_equal(s.z, np.concatenate(fresh))


def test_solution_split_and_residual_definitions(gpu):
    g = fg.build_packing(fg.PackingSpec(2))
    sol, _ = fg.run(g, fg.RunConfig(max_iterations=5))
    assert [len(v) for v in sol] == [2, 1, 2, 1]
    g = two_quadratic_graph()
    s = fg.init_state(g)
    zp = s.z.copy()
    fg.iterate(g, s)
    assert fg.residuals(g, s, zp) == pytest.approx((0.5, 1.0))
    assert s.iteration == 1


def test_seeded_init_runs_identically_on_repeat(gpu):
    """Determinism: two runs of the same state are bitwise equal (no
    atomics in any reduction)."""
    spec = fg.PackingSpec(60)
    g = fg.build_packing(spec)
    st = fg.init_state(g, seed=3)
    a = fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun"))
    b = fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun"))
    ra = fg.run(g, fg.RunConfig(max_iterations=50), state=a)[1]
    rb = fg.run(g, fg.RunConfig(max_iterations=50), state=b)[1]
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
    assert ra.history == rb.history or all(
        x[-2:] == y[-2:] for x, y in zip(ra.history, rb.history))


def test_set_edge_params_is_picked_up(gpu):
    """rho/alpha changes between runs reach the device (graph.py:232-246)."""
    spec = fg.PackingSpec(20)
    g = fg.build_packing(spec)
    st = fg.packing_init(g, spec, seed=1)
    s = fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun"))
    fg.run(g, fg.RunConfig(max_iterations=5), state=s)
    for e in (0, 7, 100):
        g.set_edge_params(e, rho=2.5, alpha=0.7)
    fg.run(g, fg.RunConfig(max_iterations=5), state=s)
    so, _h, _ = O.run(g, 5, st)      # oracle: 5 with old params...
    # replay: old params for 5, new params for 5
    g2 = fg.build_packing(spec)
    o2 = O.Oracle(g2)
    s2 = O.State.copy_of(st)
    for _ in range(5):
        o2.iterate(s2)
    for e in (0, 7, 100):
        g2.set_edge_params(e, rho=2.5, alpha=0.7)
    for _ in range(5):
        o2.iterate(s2)
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(s, k), getattr(s2, k))


def test_non_finite_output_is_located_and_named(gpu):
    b = fg.GraphBuilder()
    v = b.declare_variable(1)
    b.add_factor(fg.Quadratic([[1.0]], [1.0]), [v])
    b.add_factor(fg.NanTest("nan"), [v])
    g = b.freeze()
    with pytest.raises(RuntimeError, match=r"after x update at iteration 1: "
                                           r"edge 1 of factor 1 \(kind 'nan_test'\)"):
        fg.run(g, fg.RunConfig(max_iterations=3))
    with pytest.raises(RuntimeError, match=r"factor 1 \(kind 'nan_test'\)"):
        fg.update_x(g, fg.init_state(g))


def test_operator_failure_names_the_factor(gpu):
    b = fg.GraphBuilder()
    v = b.declare_variable(1)
    b.add_factor(fg.Quadratic([[1.0]], [1.0]), [v])
    b.add_factor(fg.NanTest("raise"), [v])
    g = b.freeze()
    with pytest.raises(RuntimeError, match=r"prox evaluation failed for factor 1 "
                                           r"\(kind 'nan_test'\)"):
        fg.run(g, fg.RunConfig(max_iterations=1))


def test_radius_weight_below_kappa_raises(gpu):
    g = fg.build_packing(fg.PackingSpec(3))
    e = int(g.factors[3].edge_range[0])          # first radius factor
    g.set_edge_params(e, rho=0.4, alpha=1.0)
    with pytest.raises(RuntimeError, match="radius prox requires rho > kappa"):
        fg.run(g, fg.RunConfig(max_iterations=1))


def test_overflow_in_z_is_reported_as_variable(gpu):
    """x and m stay finite (8.5e307 each) but three of them overflow the
    consensus sum: the failure is attributed to the z phase."""
    b = fg.GraphBuilder()
    w = b.declare_variable(1)
    v = b.declare_variable(1)
    b.add_factor(fg.Quadratic([[1.0]], [1.0]), [w])
    for _ in range(3):
        b.add_factor(fg.Quadratic([[1.7e308]], [1.0]), [v])
    g = b.freeze()
    with pytest.raises(RuntimeError,
                       match=r"non-finite value after z update at iteration 1: variable 1"):
        fg.run(g, fg.RunConfig(max_iterations=3))


def test_download_locates_first_nonfinite_entry(gpu):
    """The device records, during the download scatter, the first
    non-finite entry of each payload array in reference edge order; the
    final n check (reference engine.py:519) is built from it and must name
    the same edge a host scan of the downloaded n names."""
    from paper_1603_02526_b200 import engine
    g = fg.build_packing(fg.PackingSpec(30))
    st = fg.init_state(g, seed=1)
    P = g.total_edge_payload
    z, u, n = st.z.copy(), st.u.copy(), st.n.copy()
    rng = np.random.default_rng(0)
    picks = np.sort(rng.choice(P, 5, replace=False))
    u[picks[1:]] = -1.7e308                      # n = z - u overflows there
    z[:] = 1.7e308
    u[picks[0]] = np.nan
    plan = engine.device_plan(g)
    plan.sync(g)
    plan.upload(z, u, n)
    out = {k: np.empty(P) for k in "xmun"}
    plan.download(**out, z=np.empty(g.z_dim))
    bad = plan.nonfinite()
    for k in "xmun":
        scan = np.nonzero(~np.isfinite(out[k]))[0]
        assert bad[k] == (int(scan[0]) if scan.size else -1), k
    assert bad["u"] == picks[0] and bad["n"] == picks[0]
    msg = engine._nonfinite_message(g, None, "n", 7, first=bad["n"])
    assert msg == engine._nonfinite_message(g, out["n"], "n", 7)
    assert msg.startswith("non-finite value after n update at iteration 7: edge ")
    # a clean download resets the record
    plan.upload(st.z, st.u, st.n)
    plan.download(**out, z=np.empty(g.z_dim))
    assert plan.nonfinite() == {"x": -1, "m": -1, "u": -1, "n": -1}


# ---- operators: device batch_eval vs the reference's own outputs ----------

def _params(gd, kind):
    if kind == "mpc_dyn":
        sys_ = fg.LinearSystem(gd["mpc_dyn_A"], gd["mpc_dyn_B"])
        return {"systems": [sys_], "index": np.zeros(64, dtype=np.int64)}
    if kind == "quadratic":
        return {"targets": [gd["quadratic_p_targets0"], gd["quadratic_p_targets1"]],
                "curvatures": [gd["quadratic_p_curvatures0"], gd["quadratic_p_curvatures1"]]}
    pre = f"{kind}_p_"
    return {k[len(pre):]: gd[k] for k in gd if k.startswith(pre)}


BITWISE_KINDS = {"collision", "wall", "radius", "svm_slack", "svm_norm", "equality",
                 "mpc_cost", "mpc_init", "quadratic"}


@pytest.mark.parametrize("kind", sorted(BITWISE_KINDS | {"svm_margin", "mpc_dyn"}))
def test_device_prox_matches_reference_batch(gpu, kind):
    gd = golden("operators.npz")
    vals = [gd[f"{kind}_in{j}"] for j in range(4) if f"{kind}_in{j}" in gd]
    rhos = [gd[f"{kind}_rho{j}"] for j in range(len(vals))]
    cls = fg.operator_class(kind)
    out = cls.batch_eval(_params(gd, kind), vals, rhos)
    for j, o in enumerate(out):
        want = gd[f"{kind}_out{j}"]
        if kind in BITWISE_KINDS:
            np.testing.assert_array_equal(o, want, err_msg=f"{kind} slot {j}")
        else:
            np.testing.assert_allclose(o, want, rtol=1e-12, atol=1e-14)


def test_operator_known_answers(gpu):
    c1, r1, c2, r2 = fg.collision_prox([0.0, 0.0], 1.0, [1.0, 0.0], 1.0, 1.0, 1.0)
    np.testing.assert_array_equal(c1, [-0.25, 0.0])
    np.testing.assert_array_equal(c2, [1.25, 0.0])
    assert r1 == 0.75 and r2 == 0.75
    out = fg.Collision().eval([[0.0, 0.0], [1.0], [1.0, 0.0], [1.0]], [2.0, 2.0, 1.0, 1.0])
    np.testing.assert_allclose(out[0], [-1.0 / 6.0, 0.0])
    np.testing.assert_allclose(out[2], [1.0 + 1.0 / 3.0, 0.0])
    with pytest.warns(RuntimeWarning):
        c1, r1, c2, r2 = fg.collision_prox([0.5, 0.5], 0.4, [0.5, 0.5], 0.4, 1.0, 1.0)
    assert c1[0] != c2[0] and c1[1] == c2[1]
    assert np.linalg.norm(c1 - c2) == pytest.approx(r1 + r2)
    plane = fg.HalfPlane((0.0, 1.0), (0.0, 0.0))
    c, r = fg.wall_prox([0.3, -0.25], 0.25, plane)
    np.testing.assert_array_equal(c, [0.3, 0.0])
    assert r == 0.0
    out = fg.Wall(fg.HalfPlane((1.0, 0.0), (0.0, 0.0))).eval([[-1.0, 0.5], [1.0]], [4.0, 1.0])
    np.testing.assert_allclose(out[0], [-0.6, 0.5])
    np.testing.assert_allclose(out[1], [-0.6])
    assert fg.radius_prox(1.0, 5.0, kappa=0.5) == pytest.approx(10.0 / 9.0)
    assert fg.radius_prox(-0.3, 2.0, kappa=1.0) == pytest.approx(-0.6)
    with pytest.raises(ValueError):
        fg.Radius(1.0).eval([[1.0]], [0.5])
    x, u = fg.mpc_cost_prox([2.0, -4.0], [6.0], [1.0, 1.0], [1.0], 1.0)
    np.testing.assert_array_equal(x, [1.0, -2.0])
    np.testing.assert_array_equal(u, [3.0])
    sys_ = fg.LinearSystem([[1.0]], [[1.0]])
    x, u, x1 = fg.mpc_dyn_prox([1.0], [1.0], [2.0], sys_, 1.0, 1.0, 1.0)
    np.testing.assert_allclose(x, [2.0 / 3.0])
    np.testing.assert_allclose(u, [5.0 / 6.0])
    np.testing.assert_allclose(x1, [13.0 / 6.0])
    out = fg.MpcDyn(sys_).eval([[1.0, 1.0], [2.0, 9.0]], [1.0, 1.0])
    assert out[1][1] == 9.0
    q, u = fg.mpc_init_prox([5.0, 5.0], [3.0], [1.0, -1.0])
    np.testing.assert_array_equal(q, [1.0, -1.0])
    assert fg.svm_slack_prox(1.0, 1.0, 2.0) == 0.5
    assert fg.svm_slack_prox(-1.0, 1.0, 2.0) == 0.0
    np.testing.assert_allclose(fg.svm_norm_prox([3.0, -6.0], 1.0), [1.5, -3.0])
    point = fg.LabeledPoint([1.0, 0.0], +1)
    w, b, xi = fg.svm_margin_prox([0.0, 0.0], 0.0, 0.0, point, 1.0, 1.0, 1.0)
    np.testing.assert_allclose(w, [1.0 / 3.0, 0.0])
    assert b == pytest.approx(1.0 / 3.0) and xi == pytest.approx(1.0 / 3.0)
    a, bb = fg.equality_prox([1.0, 3.0], [3.0, 5.0], 1.0, 1.0)
    np.testing.assert_array_equal(a, [2.0, 4.0])
    np.testing.assert_array_equal(a, bb)
    op = fg.Quadratic([[1.0], [3.0]], [1.0, 3.0])
    out = op.eval([[0.0], [0.0]], [1.0, 1.0])
    assert out[0][0] == pytest.approx(0.5) and out[1][0] == pytest.approx(2.25)


@pytest.mark.parametrize("kind", sorted(BITWISE_KINDS | {"svm_margin", "mpc_dyn"}))
def test_batch_eval_matches_single_eval_bitwise(gpu, kind):
    """Reference contract (tests/test_operators.py:283-306): a factor's
    batched result equals its one-factor eval bit for bit."""
    gd = golden("operators.npz")
    vals = [gd[f"{kind}_in{j}"][:6] for j in range(4) if f"{kind}_in{j}" in gd]
    rhos = [gd[f"{kind}_rho{j}"][:6] for j in range(len(vals))]
    params = _params(gd, kind)
    cls = fg.operator_class(kind)
    sub = {}
    for k, v in params.items():
        if k == "systems":
            sub[k] = v
        elif isinstance(v, list):
            sub[k] = [a[:6] for a in v]
        else:
            sub[k] = v[:6]
    batch = cls.batch_eval(sub, vals, rhos)
    for i in range(6):
        op = cls.unstack(sub, i, tuple(v.shape[1] for v in vals))
        single = op.eval([v[i] for v in vals], [r[i] for r in rhos])
        for j, s in enumerate(single):
            np.testing.assert_array_equal(batch[j][i], s)


@pytest.mark.parametrize("name", ["pack", "svm", "mpc", "quad"])
def test_device_objective_and_violation_match_graph_helpers(gpu, name):
    """On-device objective / violation equal the host helpers (reference
    graph.py:253-263 restated per kind in operators.py)."""
    from paper_1603_02526_b200.engine import constraint_violation, objective_value
    rng = np.random.default_rng(3)
    if name == "pack":
        g = fg.build_packing(fg.PackingSpec(25))
    elif name == "svm":
        X, y = fg.gen_gaussian_arrays(60, 6, 4.0, seed=1)
        g = fg.build_svm(fg.SvmSpec.from_arrays(X, y))
    elif name == "mpc":
        g = fg.build_mpc(fg.MpcSpec(12, fg.LinearSystem(*fg.pendulum_linearization()),
                                    np.array([0.0, 0.0, 0.1, 0.0])))
    else:
        b = fg.GraphBuilder()
        v = b.declare_variable(2)
        w = b.declare_variable(1)
        b.add_factor(fg.Quadratic([[1.0, 2.0], [3.0]], [0.5, 2.0]), [v, w])
        b.add_factor(fg.Quadratic([[-1.0, 0.0]], [1.5]), [v])
        g = b.freeze()
    z = rng.normal(size=g.z_dim)
    obj = objective_value(g, z)
    vio = constraint_violation(g, z)
    assert obj == pytest.approx(g.objective_value(z), rel=1e-12, abs=1e-12)
    assert vio == pytest.approx(g.constraint_violation(z), rel=1e-12, abs=1e-13)
