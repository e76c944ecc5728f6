"""Run under torchrun (one rank per GPU): each rank runs its partition plan
of a small packing / MPC / SVM graph through ``NcclRank`` (NCCL attached,
cut partials all-gathered inside the captured iteration), the global state
is gathered, and rank 0 prints one JSON line with the max relative error
against the single-plan run.  Used by tests/test_gpu_nccl.py at world 1
(the pool gives one GPU); the same script runs unchanged at world N."""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def graph(name):
    import paper_1603_02526_b200 as fg
    if name == "pack":
        return fg.build_packing(fg.PackingSpec(150))
    if name == "mpc":
        rng = np.random.default_rng(0)
        A = 0.05 * rng.standard_normal((16, 16))
        B = 0.1 * rng.standard_normal((16, 4))
        return fg.build_mpc(fg.MpcSpec(2000, fg.LinearSystem(A, B), rng.standard_normal(16)))
    X, y = fg.gen_gaussian_arrays(3000, 32, 4.0, seed=3)
    return fg.build_svm(fg.SvmSpec.from_arrays(X, y))


def main():
    import torch.distributed as dist
    import paper_1603_02526_b200 as fg
    from paper_1603_02526_b200.distributed import NcclRank
    name, iters = sys.argv[1], int(sys.argv[2])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FG_TRANSPORT=p2p: exchange through CUDA IPC peer memory; FG_ONE_DEVICE=1
    # puts every rank on device 0 (the one-GPU pool; NCCL refuses that)
    transport = os.environ.get("FG_TRANSPORT", "nccl")
    device = 0 if os.environ.get("FG_ONE_DEVICE") == "1" else local
    if name == "lost_peer":
        # every rank attaches; only rank 0 runs: its exchange waits for the
        # other ranks' flags, gives up after the bounded wait and the run
        # fails instead of hanging
        import time
        g = graph("pack")
        st = fg.init_state(g, seed=7)
        nr = NcclRank(g, rank, world, device=device, transport=transport)
        out = {"name": name, "world": world}
        if rank == 0:
            nr.upload(st)
            t0 = time.perf_counter()
            try:
                nr.run(iters)
                out["error"] = None
            except RuntimeError as e:
                out["error"] = str(e)
            out["seconds"] = time.perf_counter() - t0
            print(json.dumps(out), flush=True)
        dist.barrier()
        dist.destroy_process_group()
        return
    if name == "pack_rank":
        from paper_1603_02526_b200.partition import packing_rank_graph
        spec = fg.PackingSpec(150)
        g = fg.build_packing(spec)
        lg = packing_rank_graph(spec, rank, world)
        st = fg.init_state(g, seed=7)
        nr = NcclRank(None, rank, world, device=device, local=lg, transport=transport)
        if world != 1:
            raise SystemExit("pack_rank check compares the gathered state at world 1 only")
        nr.upload(st)
        res, hist = nr.run(iters)
        out = fg.AdmmState(*(np.empty_like(getattr(st, k)) for k in "xmzun"))
        nr.plan.download(x=out.x, m=out.m, z=out.z, u=out.u, n=out.n)
    elif name == "mpc_rank":
        # the rank graph built from the spec alone (no global graph)
        from paper_1603_02526_b200.partition import mpc_rank_graph
        rng = np.random.default_rng(0)
        A = 0.05 * rng.standard_normal((16, 16))
        B = 0.1 * rng.standard_normal((16, 4))
        spec = fg.MpcSpec(2000, fg.LinearSystem(A, B), rng.standard_normal(16))
        g = fg.build_mpc(spec)
        lg = mpc_rank_graph(spec, rank, world)
        st = fg.init_state(g, seed=7)
        nr = NcclRank(None, rank, world, device=device, local=lg, transport=transport)
        if world != 1:
            raise SystemExit("mpc_rank check compares the gathered state at world 1 only")
        nr.upload(st)
        res, hist = nr.run(iters)
        out = fg.AdmmState(*(np.empty_like(getattr(st, k)) for k in "xmzun"))
        nr.plan.download(x=out.x, m=out.m, z=out.z, u=out.u, n=out.n)
    else:
        g = graph(name)
        st = fg.init_state(g, seed=7)
        nr = NcclRank(g, rank, world, device=device, transport=transport)
        nr.upload(st)
        res, hist = nr.run(iters)
        out = nr.gather_state(st)
    group_bitwise = None
    if rank == 0 and world > 1 and name in ("pack", "mpc", "svm"):
        # the same partition run as a local group on one device: the
        # exchange transport must not change a single bit
        from paper_1603_02526_b200.distributed import LocalGroup
        lgo, _r, _h = LocalGroup(g, world, device=device).run(iters, state=st)
        group_bitwise = all(np.array_equal(getattr(out, k), getattr(lgo, k)) for k in "xmzun")
    if rank == 0:
        single = fg.AdmmState(*(getattr(st, k).copy() for k in "xmzun"))
        _sol, rep = fg.run(g, fg.RunConfig(max_iterations=iters), state=single)
        err = {}
        for k in "xmzun":
            a, b = getattr(out, k), getattr(single, k)
            err[k] = float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))
        print(json.dumps({"name": name, "world": world, "iterations": int(res.iterations),
                          "ncut": int(getattr(nr.local, "ncut", 0)),
                          "local_edges": int(len(nr.local.edge_var)),
                          "launches": int(res.launches), "rel_err": err,
                          "transport": transport, "group_bitwise": group_bitwise,
                          "bitwise": all(np.array_equal(getattr(out, k), getattr(single, k))
                                         for k in "xmzun"),
                          "history_rows": int(len(hist))}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
