"""Temporally blocked MPC chain (csrc/fg_mpc_block.cuh): kMpcKB iterations
per launch with a recomputed halo must leave exactly the state of the
per-iteration chain (and so of the per-kind path and the reference), for
every tile/halo geometry and block/tail split; a block that meets a
failure is replayed iteration by iteration."""

import numpy as np
import pytest

from conftest import golden
import paper_1603_02526_b200 as fg
from oracle import fgadmm_oracle as O

pytestmark = pytest.mark.gpu


def _mpc(T, monkeypatch, block=True, fault=None):
    from paper_1603_02526_b200.engine import DevicePlan, _PLANS
    if block:
        monkeypatch.delenv("FGADMM_MPC_BLOCK", raising=False)
    else:
        monkeypatch.setenv("FGADMM_MPC_BLOCK", "0")
    if fault is None:
        monkeypatch.delenv("FGADMM_MPC_BLOCK_FAULT", raising=False)
    else:
        monkeypatch.setenv("FGADMM_MPC_BLOCK_FAULT", str(fault))
    gd = golden("mpc16x4_T50.npz")
    g = fg.build_mpc(fg.MpcSpec(T, fg.LinearSystem(gd["A"], gd["B"]), gd["q0"]))
    _PLANS[g] = DevicePlan(g)
    return g


def _copy(st):
    return fg.AdmmState(*(np.array(getattr(st, k), copy=True) for k in "xmzun"))


@pytest.mark.parametrize("T,K", [(40, 7), (40, 12), (300, 2), (300, 6), (300, 7),
                                 (300, 10), (300, 11), (300, 23), (5000, 31), (20011, 17),
                                 (100000, 20)])
def test_blocked_chain_bitwise_equals_per_iteration_chain(gpu, monkeypatch, T, K):
    res = []
    for block in (True, False):
        g = _mpc(T, monkeypatch, block)
        plan = fg.device_plan(g)
        st = fg.init_state(g, seed=3)
        s = _copy(st)
        _sol, rep = fg.run(g, fg.RunConfig(max_iterations=K), state=s)
        forms = plan.forms()
        assert forms["chain"] == "mpc"
        assert (forms["mpc_block"] > 0) == block
        res.append((s, rep))
    (a, ra), (b, rb) = res
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)
    np.testing.assert_allclose(np.array([r[-2:] for r in ra.history]),
                               np.array([r[-2:] for r in rb.history]), rtol=1e-12)
    assert ra.iterations == rb.iterations == K


def test_blocked_chain_within_gate_of_oracle(gpu, monkeypatch):
    g = _mpc(3000, monkeypatch)
    st = fg.init_state(g, seed=4)
    s = _copy(st)
    fg.run(g, fg.RunConfig(max_iterations=20), state=s)
    assert fg.device_plan(g).forms()["mpc_block"] > 0
    so, _h, _ = O.run(g, 20, st)
    for k in "xmzun":
        ref = getattr(so, k)
        err = np.max(np.abs(getattr(s, k) - ref)) / max(1.0, np.max(np.abs(ref)))
        assert err <= 1e-9, (k, err)


def test_blocked_chain_with_tolerances_uses_per_iteration_chain(gpu, monkeypatch):
    """A tolerance stop needs every iteration's residuals: the run stops
    at the same iteration as the unblocked run, with the same state."""
    out = []
    for block in (True, False):
        g = _mpc(200, monkeypatch, block)
        s = fg.init_state(g)
        _sol, rep = fg.run(g, fg.RunConfig(max_iterations=400000, primal_tol=1e-5,
                                           dual_tol=1e-5), state=s)
        out.append((s, rep))
    assert out[0][1].converged and out[0][1].iterations == out[1][1].iterations
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(out[0][0], k), getattr(out[1][0], k))


@pytest.mark.parametrize("fault", [2, 9, 13])
def test_failed_block_is_replayed_per_iteration(gpu, monkeypatch, fault):
    """FGADMM_MPC_BLOCK_FAULT makes the block covering that iteration
    report a failure: the run stops, the host replays from the block's
    intact input slot with the per-iteration kernels, and the result is
    bitwise the unblocked run's."""
    g = _mpc(700, monkeypatch, True, fault=fault)
    st = fg.init_state(g, seed=5)
    s = _copy(st)
    _sol, rep = fg.run(g, fg.RunConfig(max_iterations=21), state=s)
    g2 = _mpc(700, monkeypatch, False)
    s2 = _copy(st)
    _sol, rep2 = fg.run(g2, fg.RunConfig(max_iterations=21), state=s2)
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(s, k), getattr(s2, k), err_msg=k)
    assert rep.iterations == 21
    np.testing.assert_allclose(np.array([r[-2:] for r in rep.history]),
                               np.array([r[-2:] for r in rep2.history]), rtol=1e-12)
