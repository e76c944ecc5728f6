"""Multi-GPU partition logic on the CPU: partition invariants,
and the partitioned protocol (local partial sums, all-gather, rank-order
combine) checked against the single-process oracle, both in-process and
across real processes with the gloo backend (world size 2)."""

import os
import socket

import numpy as np
import pytest

import paper_1603_02526_b200 as fg
from paper_1603_02526_b200.partition import Partition, local_weight_check
from oracle import fgadmm_oracle as O


def _graphs():
    X, y = fg.gen_gaussian_arrays(40, 5, 4.0, seed=2)
    svm = fg.build_svm(fg.SvmSpec.from_arrays(X, y))
    pack = fg.build_packing(fg.PackingSpec(12))
    mpc = fg.build_mpc(fg.MpcSpec(15, fg.LinearSystem(*fg.pendulum_linearization()),
                                  np.array([0.0, 0.0, 0.1, 0.0])))
    return {"svm": svm, "pack": pack, "mpc": mpc}


@pytest.mark.parametrize("name", ["svm", "pack", "mpc"])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_partition_covers_graph_and_marks_cuts(name, world):
    g = _graphs()[name]
    part = Partition(g, world)
    locs = [part.local(r) for r in range(world)]
    edges = np.sort(np.concatenate([lg.global_edge for lg in locs]))
    np.testing.assert_array_equal(edges, np.arange(len(g.edge_var)))
    pay = np.sort(np.concatenate([lg.global_payload for lg in locs]))
    np.testing.assert_array_equal(pay, np.arange(g.total_edge_payload))
    for lg in locs:
        # local layout is the global one restricted to the rank
        np.testing.assert_array_equal(lg.global_z[lg.zmap], g.zmap[lg.global_payload])
        np.testing.assert_array_equal(lg.rho_flat, g.rho_flat[lg.global_payload])
        assert local_weight_check(lg)
        assert (lg.cut_index >= 0).sum() == np.repeat(lg.var_cut, np.diff(lg.var_offsets)).sum()
    counts = np.zeros(len(g.var_offsets) - 1, dtype=int)
    for lg in locs:
        counts[lg.global_var] += 1
    np.testing.assert_array_equal(counts > 1, part.var_cut)


def test_svm_cut_set_is_bias_plus_boundaries():
    X, y = fg.gen_gaussian_arrays(40, 5, 4.0, seed=2)
    g = fg.build_svm(fg.SvmSpec.from_arrays(X, y))
    part = Partition(g, 4)
    cut_vars = np.nonzero(part.var_cut)[0]
    assert 40 in cut_vars                     # the bias b
    assert len(cut_vars) <= 1 + 3 * 3         # plus a few per rank boundary


def _partitioned_vs_single(g, world, iters, st):
    """Run the ranks as threads in lock step (all-gather = barrier + shared
    slots) and assemble the global state."""
    import threading
    part = Partition(g, world)
    locs = [part.local(r) for r in range(world)]
    ref, ref_hist, _ = O.run(g, iters, st)
    states = [O.State(*(np.array(getattr(st, k), dtype=float)[lg.global_payload]
                        if k != "z" else np.array(st.z)[lg.global_z] for k in "xmzun"))
              for lg in locs]
    barrier = threading.Barrier(world)
    slots, lock = {}, threading.Lock()
    results = [None] * world

    def worker(r):
        counter = [0]

        def allgather(vec):
            key = counter[0]
            counter[0] += 1
            with lock:
                slots.setdefault(key, [None] * world)[r] = np.asarray(vec, dtype=float)
            barrier.wait()
            out = list(slots[key])
            barrier.wait()
            return out
        results[r] = O.run_partitioned(locs[r], iters, states[r], allgather)

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    full = O.State(*(np.zeros_like(getattr(ref, k)) for k in "xmzun"))
    for lg, (s, _h) in zip(locs, results):
        for k in "xmun":
            getattr(full, k)[lg.global_payload] = getattr(s, k)
        full.z[lg.global_z] = s.z
    return ref, ref_hist, full, results[0][1]


@pytest.mark.parametrize("name", ["svm", "pack", "mpc"])
@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_protocol_matches_single_process(name, world):
    g = _graphs()[name]
    st = fg.init_state(g, seed=4)
    ref, ref_hist, full, hist = _partitioned_vs_single(g, world, 12, st)
    for k in "xmzun":
        a, b = getattr(full, k), getattr(ref, k)
        assert np.max(np.abs(a - b)) <= 1e-12 * max(1.0, np.max(np.abs(b))), k
    np.testing.assert_allclose(np.array(hist), np.array(ref_hist), rtol=1e-10)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_rank(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = _graphs()["svm"]
    st = fg.init_state(g, seed=4)
    part = Partition(g, world)
    lg = part.local(rank)
    ls = O.State(*(np.array(getattr(st, k))[lg.global_payload] if k != "z"
                   else np.array(st.z)[lg.global_z] for k in "xmzun"))

    def ag(vec):
        t = torch.as_tensor(np.asarray(vec, dtype=np.float64))
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t)
        return [o.numpy() for o in outs]

    s, hist = O.run_partitioned(lg, 12, ls, ag)
    parts = [None] * world
    dist.all_gather_object(parts, (rank, {k: getattr(s, k) for k in "xmzun"}, hist))
    if rank == 0:
        np.savez(out_path, **{f"{r}_{k}": v for r, arrs, _h in parts for k, v in arrs.items()},
                 hist=np.array(parts[0][2]))
    dist.destroy_process_group()


def test_gloo_world2_partitioned_svm_matches_single(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    out = str(tmp_path / "res.npz")
    mp.spawn(_gloo_rank, args=(world, _free_port(), out), nprocs=world, join=True)
    g = _graphs()["svm"]
    st = fg.init_state(g, seed=4)
    ref, ref_hist, _ = O.run(g, 12, st)
    res = np.load(out)
    part = Partition(g, world)
    full = {k: np.zeros_like(getattr(ref, k)) for k in "xmzun"}
    for r in range(world):
        lg = part.local(r)
        for k in "xmun":
            full[k][lg.global_payload] = res[f"{r}_{k}"]
        full["z"][lg.global_z] = res[f"{r}_z"]
    for k in "xmzun":
        np.testing.assert_allclose(full[k], getattr(ref, k), rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(res["hist"], np.array(ref_hist), rtol=1e-10)


def test_svm_rank_graph_equals_partition_local():
    """The per-rank SVM builder (weak-scaled multi-GPU runs) emits exactly
    the partitioner's local graph when the partition splits at the ranks'
    point blocks (world 2, equal blocks)."""
    from paper_1603_02526_b200.partition import Partition, svm_rank_graph
    n, world = 1200, 2
    Xs, ys = zip(*[fg.gen_gaussian_arrays(n, 32, 4.0, seed=r) for r in range(world)])
    g = fg.build_svm(fg.SvmSpec.from_arrays(np.concatenate(Xs), np.concatenate(ys)))
    part = Partition(g, world)
    for r in range(world):
        lg, rg = part.local(r), svm_rank_graph(Xs[r], ys[r], r, world)
        for k in ("edge_var", "edge_offsets", "var_offsets", "edge_rho", "z_weights",
                  "cut_index"):
            np.testing.assert_array_equal(np.asarray(getattr(lg, k)), np.asarray(getattr(rg, k)),
                                          err_msg=k)
        assert lg.ncut == rg.ncut
        for (c1, d1, _f1, v1, p1), (c2, d2, _f2, v2, p2) in zip(lg.blocks, rg.blocks):
            assert c1.kind == c2.kind and tuple(d1) == tuple(d2)
            np.testing.assert_array_equal(v1, v2)
            for k in p1:
                np.testing.assert_array_equal(np.asarray(p1[k]), np.asarray(p2[k]))


def _gloo_rank_graph(rank, world, port, out_path, n):
    import torch
    import torch.distributed as dist
    from paper_1603_02526_b200.partition import svm_rank_graph
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, y = fg.gen_gaussian_arrays(n, 8, 4.0, seed=20 + rank)
    lg = svm_rank_graph(X, y, rank, world)          # no global graph on this rank
    st = fg.init_state(lg, seed=None)
    ls = O.State(*(np.array(getattr(st, k)) for k in "xmzun"))

    def ag(vec):
        t = torch.as_tensor(np.asarray(vec, dtype=np.float64))
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t)
        return [o.numpy() for o in outs]

    s, hist = O.run_partitioned(lg, 10, ls, ag)
    parts = [None] * world
    dist.all_gather_object(parts, (rank, s.z, hist))
    if rank == 0:
        np.savez(out_path, **{f"z{r}": z for r, z, _h in parts}, hist=np.array(parts[0][2]))
    dist.destroy_process_group()


def test_gloo_world2_rank_graphs_match_single(tmp_path):
    """Weak-scaled protocol over gloo: each process builds only its rank
    graph from its own points; the exchanged run equals the single-process
    oracle on the concatenated SVM."""
    import torch.multiprocessing as mp
    world, n = 2, 300
    out = str(tmp_path / "rg.npz")
    mp.spawn(_gloo_rank_graph, args=(world, _free_port(), out, n), nprocs=world, join=True)
    Xs, ys = zip(*[fg.gen_gaussian_arrays(n, 8, 4.0, seed=20 + r) for r in range(world)])
    g = fg.build_svm(fg.SvmSpec.from_arrays(np.concatenate(Xs), np.concatenate(ys)))
    ref, ref_hist, _ = O.run(g, 10, fg.init_state(g))
    res = np.load(out)
    D, N = 8, n * world
    for r in range(world):
        z = res[f"z{r}"]
        np.testing.assert_allclose(z[:n * D], ref.z[r * n * D:(r + 1) * n * D], rtol=1e-11,
                                   atol=1e-13)
        nb = n * D + (0 if r == world - 1 else D)
        np.testing.assert_allclose(z[nb], ref.z[N * D], rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(res["hist"], np.array(ref_hist), rtol=1e-10)


def test_local_graph_follows_set_edge_params():
    """A rank's LocalGraph re-slices rho, alpha and the z weights when the
    global graph's parameters change (its param_version moves), so device
    plans of partitioned runs re-sync instead of keeping stale weights."""
    import paper_1603_02526_b200 as fg
    from paper_1603_02526_b200.partition import Partition
    g = fg.build_packing(fg.PackingSpec(12))
    part = Partition(g, 2)
    lg = part.local(1)
    v0 = lg.param_version
    e = int(lg.global_edge[3])
    g.set_edge_params(e, rho=2.5, alpha=0.75)
    assert lg.param_version != v0
    assert lg.edge_rho[3] == 2.5 and lg.edge_alpha[3] == 0.75
    np.testing.assert_array_equal(lg.z_weights, g.z_weights[lg.global_z])
    np.testing.assert_array_equal(lg.rho_flat, np.repeat(lg.edge_rho, np.diff(lg.edge_offsets)))


@pytest.mark.parametrize("T,world", [(2, 2), (5, 3), (40, 4), (333, 8), (100, 2)])
def test_mpc_rank_graph_equals_partition_local(T, world):
    """The per-rank MPC builder (no global graph on the host) emits exactly
    the partitioner's local graph: variables, factors in creation order,
    parameters, global z weights (rho != 1) and the canonical cut vector."""
    from paper_1603_02526_b200.partition import Partition, mpc_rank_graph
    rng = np.random.default_rng(0)
    A, B = 0.05 * rng.standard_normal((4, 4)), 0.1 * rng.standard_normal((4, 2))
    spec = fg.MpcSpec(T, fg.LinearSystem(A, B), rng.standard_normal(4), rho=1.5, alpha=0.8)
    part = Partition(fg.build_mpc(spec), world)
    for r in range(world):
        lg = part.local(r)
        if len(lg.edge_var) == 0:
            with pytest.raises(ValueError):
                mpc_rank_graph(spec, r, world)
            continue
        rg = mpc_rank_graph(spec, r, world)
        for k in ("edge_var", "edge_offsets", "var_offsets", "edge_rho", "edge_alpha",
                  "z_weights", "cut_index"):
            np.testing.assert_array_equal(np.asarray(getattr(lg, k)), np.asarray(getattr(rg, k)),
                                          err_msg=k)
        assert lg.ncut == rg.ncut
        assert len(lg.blocks) == len(rg.blocks)
        for (c1, d1, _f1, v1, p1), (c2, d2, _f2, v2, p2) in zip(lg.blocks, rg.blocks):
            assert c1.kind == c2.kind and tuple(d1) == tuple(d2)
            np.testing.assert_array_equal(v1, v2)
            for k in p1:
                if k != "systems":
                    np.testing.assert_array_equal(np.asarray(p1[k]), np.asarray(p2[k]))


@pytest.mark.parametrize("N,world", [(1, 2), (2, 3), (7, 4), (40, 3), (151, 8), (64, 7)])
def test_packing_rank_graph_equals_partition_local(N, world):
    """The per-rank packing builder (no global graph on the host) emits
    exactly the partitioner's local graph -- including ranks whose boundary
    falls between a disk's center and its radius -- and packing_init on it
    is the scatter of the global packing_init state."""
    from paper_1603_02526_b200.partition import Partition, packing_rank_graph
    spec = fg.PackingSpec(N, rho=1.5, rho_radius=3.0, alpha=0.7)
    g = fg.build_packing(spec)
    part = Partition(g, world)
    st = fg.packing_init(g, spec, seed=0) if N > 1 else None
    for r in range(world):
        lg = part.local(r)
        if len(lg.edge_var) == 0:
            with pytest.raises(ValueError):
                packing_rank_graph(spec, r, world)
            continue
        rg = packing_rank_graph(spec, r, world)
        for k in ("edge_var", "edge_offsets", "var_offsets", "edge_rho", "edge_alpha",
                  "z_weights", "cut_index"):
            np.testing.assert_array_equal(np.asarray(getattr(lg, k)), np.asarray(getattr(rg, k)),
                                          err_msg=k)
        assert lg.ncut == rg.ncut
        assert len(lg.blocks) == len(rg.blocks)
        for (c1, d1, _f1, v1, p1), (c2, d2, _f2, v2, p2) in zip(lg.blocks, rg.blocks):
            assert c1.kind == c2.kind and tuple(d1) == tuple(d2)
            np.testing.assert_array_equal(v1, v2)
            for k in p1:
                np.testing.assert_array_equal(np.asarray(p1[k]), np.asarray(p2[k]))
        if st is not None:
            rs = fg.packing_init(rg, spec, seed=0)
            np.testing.assert_array_equal(np.asarray(st.z)[lg.global_z], rs.z)
            np.testing.assert_array_equal(np.asarray(st.n)[lg.global_payload], rs.n)
