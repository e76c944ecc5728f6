"""The fused SVM-chain kernel (csrc/fg_chain.cuh) against the generic
per-kind path and the CPU oracle.

The chain kernel evaluates every factor touching w_i / xi_i and finishes
their z and u updates in one pass; its arithmetic is the per-kind kernels'
operation by operation, so the two device paths must agree BITWISE, and
both match the oracle (reference engine.py + operators.py) within the
SVM tolerance (1e-9 relative, 32-term margin dots)."""

import numpy as np
import pytest

import paper_1603_02526_b200 as fg
from oracle import fgadmm_oracle as O
from paper_1603_02526_b200.engine import DevicePlan, _PLANS

pytestmark = pytest.mark.gpu

REL = 1e-9


def copy(st):
    return fg.AdmmState(*(np.array(getattr(st, k), copy=True) for k in "xmzun"),
                        iteration=st.iteration)


def svm_graph(n, dim=32, seed=0):
    X, y = fg.gen_gaussian_arrays(n, dim, 4.0, seed=seed)
    return fg.build_svm(fg.SvmSpec.from_arrays(X, y))


def plan_for(g, monkeypatch, chain):
    if chain:
        monkeypatch.delenv("FGADMM_NO_CHAIN", raising=False)
    else:
        monkeypatch.setenv("FGADMM_NO_CHAIN", "1")
    _PLANS[g] = DevicePlan(g)
    assert _PLANS[g].info["fused_chain"] == chain
    return _PLANS[g]


def run_both(g, st, monkeypatch, cfgs):
    """The same sequence of run() calls on the chain and the generic path."""
    out = []
    for chain in (True, False):
        plan_for(g, monkeypatch, chain)
        s = copy(st)
        reps = [fg.run(g, cfg, state=s)[1] for cfg in cfgs]
        out.append((s, reps))
    return out


@pytest.mark.parametrize("n,dim,iters", [(33, 32, 7), (200, 32, 10), (5000, 32, 12),
                                         (40_000, 32, 5), (300, 7, 9), (100, 1, 6)])
def test_chain_bitwise_equals_generic(gpu, monkeypatch, n, dim, iters):
    g = svm_graph(n, dim, seed=n)
    st = fg.init_state(g, seed=3)
    (sc, rc), (sg, rg) = run_both(g, st, monkeypatch, [fg.RunConfig(max_iterations=iters)])
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(sc, k), getattr(sg, k), err_msg=k)
    assert rc[0].iterations == rg[0].iterations == iters
    assert rc[0].kernel_launches < rg[0].kernel_launches


@pytest.mark.parametrize("env", [{}, {"FGADMM_CHAIN_NO_UNIT": "1"}, {"FGADMM_CHAIN_GENERIC": "1"}])
def test_chain_forms_bitwise(gpu, monkeypatch, env):
    """Every form of the chain on unit weights (unit, weighted, generic)
    equals the per-kind path bitwise."""
    g = svm_graph(20_000, 32, seed=9)
    st = fg.init_state(g, seed=2)
    outs = []
    for chain in (True, False):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        plan_for(g, monkeypatch, chain)
        s = copy(st)
        fg.run(g, fg.RunConfig(max_iterations=11), state=s)
        if chain:
            want = {"FGADMM_CHAIN_NO_UNIT": "fast", "FGADMM_CHAIN_GENERIC": "generic"}
            assert _PLANS[g].chain_form() == next((want[k] for k in env), "unit")
        outs.append(s)
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(outs[0], k), getattr(outs[1], k), err_msg=k)


def test_chain_matches_oracle(gpu, monkeypatch):
    g = svm_graph(3000, 32, seed=11)
    plan_for(g, monkeypatch, True)
    st = fg.init_state(g, seed=5)
    s = copy(st)
    fg.run(g, fg.RunConfig(max_iterations=9), state=s)
    so, _h, _ = O.run(g, 9, st)
    for k in "xmzun":
        a, b = getattr(s, k), getattr(so, k)
        scale = max(1.0, float(np.max(np.abs(b))))
        assert float(np.max(np.abs(a - b))) <= REL * scale, k


def test_chain_resume_and_odd_chunks(gpu, monkeypatch):
    """Runs of 1, 2, 5 and 17 iterations (graph chunks + tail) resumed from
    the downloaded state equal one 25-iteration run."""
    g = svm_graph(700, 32, seed=2)
    st = fg.init_state(g, seed=9)
    plan_for(g, monkeypatch, True)
    a = copy(st)
    for k in (1, 2, 5, 17):
        fg.run(g, fg.RunConfig(max_iterations=k), state=a)
    b = copy(st)
    fg.run(g, fg.RunConfig(max_iterations=25), state=b)
    assert a.iteration == b.iteration == 25
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)


def test_chain_tolerance_stop_and_history(gpu, monkeypatch):
    g = svm_graph(500, 32, seed=4)
    st = fg.init_state(g)
    cfg = fg.RunConfig(max_iterations=20000, primal_tol=1e-3, dual_tol=1e-3, record_every=50)
    (sc, rc), (sg, rg) = run_both(g, st, monkeypatch, [cfg])
    assert rc[0].converged and rg[0].converged
    assert rc[0].iterations == rg[0].iterations < 20000
    hc = np.array([h[-2:] for h in rc[0].history])
    hg = np.array([h[-2:] for h in rg[0].history])
    np.testing.assert_allclose(hc, hg, rtol=1e-12, atol=0)
    np.testing.assert_array_equal(sc.z, sg.z)


def test_chain_error_message_equals_generic(gpu, monkeypatch):
    """A state that overflows after the first iteration: both paths raise
    the reference's message for the same (iteration, phase, culprit)."""
    g = svm_graph(64, 32, seed=7)
    st = fg.init_state(g, seed=1)
    st.u[::97] = 1.7e308
    st.n[:] = 0.0
    msgs = []
    for chain in (True, False):
        plan_for(g, monkeypatch, chain)
        s = copy(st)
        with pytest.raises(RuntimeError) as ei:
            fg.run(g, fg.RunConfig(max_iterations=20), state=s)
        msgs.append((str(ei.value), s.iteration))
    assert msgs[0] == msgs[1]


def test_chain_profile_labels(gpu, monkeypatch):
    g = svm_graph(2000, 32)
    plan = plan_for(g, monkeypatch, True)
    st = fg.init_state(g)
    plan.sync(g)
    plan.upload(st.z, st.u, st.n)
    prof = plan.profile_kernels(4)
    assert "chain_svm" in prof and prof["chain_svm"][1] == 2     # iteration 2 untimed (warm pass)
    assert not any(k.startswith("edge_") for k in prof)


@pytest.mark.parametrize("rho,alpha", [(2.0, 1.0), (0.5, 1.3), (1.0, 1.5), (0.7, 1.3)])
def test_chain_general_weights_bitwise(gpu, monkeypatch, rho, alpha):
    """Non-unit weights take the weighted form (weights loaded per point,
    per-point division tables); it stays bitwise equal to the per-kind
    path."""
    X, y = fg.gen_gaussian_arrays(3000, 32, 4.0, seed=12)
    g = fg.build_svm(fg.SvmSpec.from_arrays(X, y, rho=rho, alpha=alpha))
    st = fg.init_state(g, seed=6)
    (sc, _), (sg, _) = run_both(g, st, monkeypatch, [fg.RunConfig(max_iterations=8)])
    plan_for(g, monkeypatch, True).sync(g)
    forms = _PLANS[g].forms()
    # one rho and one alpha everywhere: the weight lanes read the 4-double
    # uniform table (unit weights take the unit form instead)
    assert forms["chain"] == "fast" and forms["chain_uniform"]
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(sc, k), getattr(sg, k), err_msg=k)


def test_chain_random_edge_weights_bitwise_and_oracle(gpu, monkeypatch):
    """Every edge its own rho and alpha (set_edge_params on a sample, the
    three-weight use case of PAPER.md:130): the weighted chain is bitwise the
    per-kind path and within 1e-9 of the oracle."""
    X, y = fg.gen_gaussian_arrays(1500, 32, 4.0, seed=21)
    g = fg.build_svm(fg.SvmSpec.from_arrays(X, y, rho=1.3, alpha=0.9))
    rng = np.random.default_rng(4)
    for e in rng.choice(len(g.edge_var), 3000, replace=False):
        g.set_edge_params(int(e), float(rng.uniform(0.3, 3.0)), float(rng.uniform(0.5, 1.7)))
    st = fg.init_state(g, seed=8)
    (sc, _), (sg, _) = run_both(g, st, monkeypatch, [fg.RunConfig(max_iterations=9)])
    plan_for(g, monkeypatch, True).sync(g)
    assert _PLANS[g].chain_form() == "fast" and not _PLANS[g].forms()["chain_uniform"]
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(sc, k), getattr(sg, k), err_msg=k)
    so, _h, _ = O.run(g, 9, st)
    for k in "xmzun":
        a, b = getattr(sc, k), getattr(so, k)
        assert float(np.max(np.abs(a - b))) <= REL * max(1.0, float(np.max(np.abs(b)))), k


def test_chain_unit_form_follows_set_edge_params(gpu, monkeypatch):
    """A run with unit weights, then one edge re-weighted (the plan leaves the
    unit-weight form), then restored: every run bitwise equal to the
    per-kind path on the same sequence of weights."""
    g = svm_graph(2500, 32, seed=13)
    st = fg.init_state(g, seed=2)
    e = int(np.flatnonzero(g.edge_var == g.edge_var[0])[0])

    def seq(chain):
        plan_for(g, monkeypatch, chain)
        s = copy(st)
        g.set_edge_params(e, 1.0, 1.0)
        fg.run(g, fg.RunConfig(max_iterations=4), state=s)
        g.set_edge_params(e, 3.0, 0.5)
        fg.run(g, fg.RunConfig(max_iterations=5), state=s)
        g.set_edge_params(e, 1.0, 1.0)
        fg.run(g, fg.RunConfig(max_iterations=3), state=s)
        return s

    a, b = seq(True), seq(False)
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)
