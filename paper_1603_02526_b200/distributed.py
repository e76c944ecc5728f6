"""Multi-GPU execution of one graph.

``LocalGroup`` runs the G partition plans of one graph on ONE device and
exchanges the cut partial sums with device copies: it validates the
partitioned algorithm on a single GPU against the one-plan result.

``NcclRank`` is the production path: one process per GPU (torchrun), each
rank builds the same graph (or only its part: partition.*_rank_graph),
keeps its own partition plan, and the plans all-gather the cut partials
and residual partials inside the CUDA-graph-captured iteration -- with
NCCL (``transport="nccl"``) or by storing them straight into the peers'
receive buffers over NVLink with epoch flags (``transport="p2p"``, CUDA
IPC handles exchanged once through ``torch.distributed``).  ``torch.distributed`` only broadcasts the
NCCL unique id and (for ``gather_state``) moves host arrays.

Parity: non-cut variables are summed exactly as on one GPU; a cut
variable's z is the rank-order sum of per-rank NumPy-tree partials, which
agrees with the single-GPU tree to ~1e-15 relative (bound 1e-9).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _native
from .engine import AdmmState, DevicePlan, init_state
from .partition import Partition


def nccl_library():
    """Path of the libnccl.so.2 bundled with torch (None: default search)."""
    try:
        import nvidia.nccl as _n
        for base in _n.__path__:
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                return cand
    except ImportError:
        pass
    return None


def _scatter_local(lg, state):
    """A rank's local state from the global one."""
    P = lg.global_payload
    return AdmmState(x=state.x[P].copy(), m=state.m[P].copy(), z=state.z[lg.global_z].copy(),
                     u=state.u[P].copy(), n=state.n[P].copy(), iteration=state.iteration)


def _gather_into(lg, local, state):
    P = lg.global_payload
    for k in ("x", "m", "u", "n"):
        getattr(state, k)[P] = getattr(local, k)
    state.z[lg.global_z] = local.z


class LocalGroup:
    """All partition plans of ``graph`` on one device (validation path)."""

    def __init__(self, graph, world, device=None):
        self.graph = graph
        self.part = Partition(graph, world)
        self.locals = [self.part.local(r) for r in range(world)]
        self.plans = [DevicePlan(lg, device=device) for lg in self.locals]

    def run(self, iterations, state=None, primal_tol=0.0, dual_tol=0.0):
        g = self.graph
        st = state if state is not None else init_state(g)
        for lg, plan in zip(self.locals, self.plans):
            plan.sync(lg)
            ls = _scatter_local(lg, st)
            plan.upload(ls.z, ls.u, ls.n)
        cfg = _native.RunConfig()
        cfg.max_iterations = int(iterations)
        cfg.primal_tol = float(primal_tol)
        cfg.dual_tol = float(dual_tol)
        cfg.first_reads_n = 1
        res = _native.RunResult()
        hist = np.zeros(2 * int(iterations))
        handles = (C.c_void_p * len(self.plans))(*[p._h.value for p in self.plans])
        lib = _native.load()
        _native.check(lib.fg_group_run(handles, len(self.plans), C.byref(cfg),
                                       _native.dptr(hist), C.byref(res)))
        out = AdmmState(*(np.array(getattr(st, k), dtype=float, copy=True) for k in "xmzun"),
                        iteration=st.iteration + int(res.iterations))
        for lg, plan in zip(self.locals, self.plans):
            ls = AdmmState(*(np.empty(lg.total_edge_payload) for _ in range(2)),
                           np.empty(lg.z_dim),
                           *(np.empty(lg.total_edge_payload) for _ in range(2)))
            plan.download(x=ls.x, m=ls.m, z=ls.z, u=ls.u, n=ls.n)
            _gather_into(lg, ls, out)
        return out, res, hist.reshape(-1, 2)[:res.iterations]


def group_run_locals(graphs, iterations, device=None):
    """Run already-partitioned rank graphs (e.g. ``svm_rank_graph``) as a
    local group on one device from their zero states; returns the per-rank
    downloaded states and the run result.  The validation path of the
    weak-scaled multi-GPU benchmark."""
    plans = [DevicePlan(lg, device=device) for lg in graphs]
    for lg, plan in zip(graphs, plans):
        plan.sync(lg)
        st = init_state(lg)
        plan.upload(st.z, st.u, st.n)
    cfg = _native.RunConfig()
    cfg.max_iterations = int(iterations)
    cfg.first_reads_n = 1
    res = _native.RunResult()
    hist = np.zeros(2 * int(iterations))
    handles = (C.c_void_p * len(plans))(*[p._h.value for p in plans])
    _native.check(_native.load().fg_group_run(handles, len(plans), C.byref(cfg),
                                              _native.dptr(hist), C.byref(res)))
    outs = []
    for lg, plan in zip(graphs, plans):
        ls = AdmmState(*(np.empty(lg.total_edge_payload) for _ in range(2)), np.empty(lg.z_dim),
                       *(np.empty(lg.total_edge_payload) for _ in range(2)))
        plan.download(x=ls.x, m=ls.m, z=ls.z, u=ls.u, n=ls.n)
        outs.append(ls)
    return outs, res, plans


class NcclRank:
    """This process's partition plan of ``graph``, exchanging over NCCL.

    ``group`` is an initialised ``torch.distributed`` process group (any
    backend); it carries the NCCL unique id and host-side gathers only.
    ``local`` (instead of ``graph``) is an already-built rank graph with
    ``cut_index`` / ``ncut`` (``partition.svm_rank_graph``): no global
    graph is built on the host.
    """

    def __init__(self, graph, rank, world, group=None, device=None, local=None,
                 transport="nccl"):
        import torch.distributed as dist
        self.graph = graph
        self.rank, self.world = int(rank), int(world)
        if local is None:
            self.part = Partition(graph, world)
            self.local = self.part.local(self.rank)
        else:
            self.part = None
            self.local = local
        self.plan = DevicePlan(self.local, device=device)
        self.transport = transport
        lib = _native.load()
        if transport == "p2p":
            # peer memory: export this rank's receive buffer and flags as
            # CUDA IPC handles, all-gather them, attach the peers'
            h = C.create_string_buffer(128)
            _native.check(lib.fg_p2p_export(self.plan._h, self.world, h))
            allh = [None] * self.world
            dist.all_gather_object(allh, bytes(h.raw), group=group)
            pay = [None] * self.world
            dist.all_gather_object(pay, int(self.local.total_edge_payload), group=group)
            buf = C.create_string_buffer(b"".join(allh), 128 * self.world)
            _native.check(lib.fg_plan_attach_p2p(self.plan._h, self.rank, self.world, buf,
                                                 int(sum(pay))))
            dist.barrier(group=group)              # every rank attached before any run
        elif transport == "nccl":
            path = nccl_library()
            bpath = path.encode() if path else None
            uid = C.create_string_buffer(128)
            if self.rank == 0:
                _native.check(lib.fg_nccl_unique_id(bpath, uid))
            obj = [bytes(uid.raw) if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            _native.check(lib.fg_plan_attach_nccl(self.plan._h, bpath, obj[0], self.rank,
                                                  self.world))
        else:
            raise ValueError(f"unknown transport {transport!r}")
        self._dist = dist
        self._group = group

    def upload(self, state):
        """``state``: the global state, or (rank graphs) this rank's own."""
        lg = self.local
        self.plan.sync(lg)
        ls = _scatter_local(lg, state) if self.part is not None else state
        self.plan.upload(ls.z, ls.u, ls.n)

    def run(self, iterations, primal_tol=0.0, dual_tol=0.0, graph_chunk=16):
        return self.plan.run(iterations, primal_tol, dual_tol, graph_chunk=graph_chunk)

    def gather_state(self, like):
        """Assemble the global state on every rank (host all-gather)."""
        lg = self.local
        ls = AdmmState(*(np.empty(lg.total_edge_payload) for _ in range(2)), np.empty(lg.z_dim),
                       *(np.empty(lg.total_edge_payload) for _ in range(2)))
        self.plan.download(x=ls.x, m=ls.m, z=ls.z, u=ls.u, n=ls.n)
        parts = [None] * self.world
        self._dist.all_gather_object(parts, (self.rank, {k: getattr(ls, k) for k in "xmzun"}),
                                     group=self._group)
        out = AdmmState(*(np.array(getattr(like, k), dtype=float, copy=True) for k in "xmzun"),
                        iteration=like.iteration)
        for r, arrs in parts:
            lgr = self.part.local(r) if r != self.rank else lg
            _gather_into(lgr, AdmmState(**arrs), out)
        return out
