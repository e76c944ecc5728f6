"""Partitioned (multi-GPU) device algorithm validated on one GPU: the G
partition plans of a graph run as a local group (cut partials exchanged by
device copies, same kernels and exchange points as the NCCL path) and must
match the single-plan run and the partitioned oracle (1e-9 relative)."""

import numpy as np
import pytest

import paper_1603_02526_b200 as fg
from paper_1603_02526_b200.distributed import LocalGroup
from oracle import fgadmm_oracle as O

pytestmark = pytest.mark.gpu


def _graph(name):
    if name == "svm":
        X, y = fg.gen_gaussian_arrays(3000, 32, 4.0, seed=3)
        return fg.build_svm(fg.SvmSpec.from_arrays(X, y))
    if name == "pack":
        return fg.build_packing(fg.PackingSpec(150))
    return fg.build_mpc(fg.MpcSpec(400, fg.LinearSystem(*fg.pendulum_linearization()),
                                   np.array([0.0, 0.0, 0.1, 0.0])))


def _close(a, b, rel=1e-9):
    scale = max(1.0, float(np.max(np.abs(b))))
    return float(np.max(np.abs(a - b))) <= rel * scale


@pytest.mark.parametrize("name", ["svm", "pack", "mpc"])
@pytest.mark.parametrize("world", [2, 4])
def test_local_group_matches_single_plan(gpu, name, world):
    g = _graph(name)
    st = fg.init_state(g, seed=7)
    single = fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun"))
    _sol, rep = fg.run(g, fg.RunConfig(max_iterations=15), state=single)
    grp = LocalGroup(g, world)
    assert grp.part.ncut > 0
    out, res, hist = grp.run(15, st)
    assert res.iterations == 15 and res.error_phase == -1
    for k in "xmzun":
        assert _close(getattr(out, k), getattr(single, k)), k
    np.testing.assert_allclose(hist, np.array([r[-2:] for r in rep.history]), rtol=1e-9)


def test_local_group_tolerance_stop_matches_single(gpu):
    g = fg.build_mpc(fg.MpcSpec(10, fg.LinearSystem(*fg.pendulum_linearization()),
                                np.array([0.0, 0.0, 0.1, 0.0])))
    st = fg.init_state(g)
    _sol, rep = fg.run(g, fg.RunConfig(max_iterations=20000, primal_tol=1e-7, dual_tol=1e-7),
                       state=fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun")))
    assert rep.converged
    out, res, _h = LocalGroup(g, 3).run(20000, st, primal_tol=1e-7, dual_tol=1e-7)
    assert res.converged
    assert abs(int(res.iterations) - rep.iterations) <= 1


def test_local_group_matches_partitioned_oracle_bitwise_on_noncut(gpu):
    """Variables that are not cut are finished exactly as on one GPU, so a
    packing partition agrees with the partitioned oracle to rounding of
    the cut sums only."""
    g = _graph("pack")
    st = fg.init_state(g, seed=2)
    grp = LocalGroup(g, 2)
    out, _res, _h = grp.run(5, st)
    ref, _rh, _ = O.run(g, 5, st)
    for k in "xmzun":
        assert _close(getattr(out, k), getattr(ref, k)), k


@pytest.mark.parametrize("world", [2, 3])
def test_svm_partition_runs_fused_chain_bitwise_vs_per_kind(gpu, monkeypatch, world):
    """Partition plans of the SVM chain keep the fused chain kernel (cut
    weight copies and the bias go through the exchange); the result is
    bitwise the per-kind partitioned run and within 1e-9 of one plan."""
    X, y = fg.gen_gaussian_arrays(2400, 32, 4.0, seed=5)
    g = fg.build_svm(fg.SvmSpec.from_arrays(X, y))
    st = fg.init_state(g, seed=4)
    outs = []
    for chain in (True, False):
        if chain:
            monkeypatch.delenv("FGADMM_NO_CHAIN", raising=False)
        else:
            monkeypatch.setenv("FGADMM_NO_CHAIN", "1")
        grp = LocalGroup(g, world)
        assert all(p.info["fused_chain"] == chain for p in grp.plans)
        out, res, hist = grp.run(12, st)
        assert res.iterations == 12 and res.error_phase == -1
        outs.append((out, hist))
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(outs[0][0], k), getattr(outs[1][0], k), err_msg=k)
    single = fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun"))
    fg.run(g, fg.RunConfig(max_iterations=12), state=single)
    for k in "xmzun":
        assert _close(getattr(outs[0][0], k), getattr(single, k)), k


@pytest.mark.parametrize("world", [2, 4])
def test_svm_rank_graphs_match_single_plan(gpu, world):
    """Weak-scaled multi-GPU path: rank graphs built directly from each
    rank's points (partition.svm_rank_graph), run as a group with the cut
    exchange, agree with one plan of the concatenated SVM (1e-9)."""
    from paper_1603_02526_b200.distributed import group_run_locals
    from paper_1603_02526_b200.partition import svm_rank_graph
    n, D = 700, 32
    Xs, ys = zip(*[fg.gen_gaussian_arrays(n, D, 4.0, seed=10 + r) for r in range(world)])
    g = fg.build_svm(fg.SvmSpec.from_arrays(np.concatenate(Xs), np.concatenate(ys)))
    single = fg.init_state(g)
    fg.run(g, fg.RunConfig(max_iterations=10), state=single)
    graphs = [svm_rank_graph(Xs[r], ys[r], r, world) for r in range(world)]
    outs, res, plans = group_run_locals(graphs, 10)
    assert res.iterations == 10 and res.error_phase == -1
    assert all(p.chain_form() in ("unit", "fast") for p in plans)
    N = n * world
    for r, ls in enumerate(outs):
        wz = ls.z[:n * D]
        assert _close(wz, single.z[r * n * D:(r + 1) * n * D]), r
        nb = n * D + (0 if r == world - 1 else D)
        assert _close(ls.z[nb:nb + 1], single.z[N * D:N * D + 1])
        assert _close(ls.z[nb + 1:], single.z[N * D + 1 + r * n:N * D + 1 + (r + 1) * n])


@pytest.mark.parametrize("name", ["svm", "pack"])
def test_local_group_reads_n_per_plan(gpu, name):
    """Whether iteration 1 reads the uploaded n is decided per plan: with n
    edited on one rank's payload only (every other rank's n equals z - u,
    so those plans may start on their chain forms), the group still reads
    the edited n there and matches one plan run from the same state."""
    g = _graph(name)
    st = fg.init_state(g, seed=6)
    grp = LocalGroup(g, 2)
    P1 = grp.locals[1].global_payload
    rng = np.random.default_rng(1)
    st.n[P1[:50]] += rng.uniform(-0.1, 0.1, 50)
    single = fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun"))
    fg.run(g, fg.RunConfig(max_iterations=6), state=single)
    out, res, _h = grp.run(6, st)
    assert res.iterations == 6
    for k in "xmzun":
        assert _close(getattr(out, k), getattr(single, k)), k
