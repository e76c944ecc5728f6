"""Factor partitioning for multi-GPU runs.

Each rank owns a subset of the factors and all of their edges, so the edge
pass (prox) is purely local.  A variable whose incident edges live on more
than one rank is *cut*: every rank sums its own part of the variable's
consensus segment (``m * rho`` over its local edges, in creation order),
the partial sums are all-gathered and added in rank order, and every rank
finalises the same z and updates its local u.  Non-cut variables are
finished locally, exactly as on one GPU.

Assignment: a factor goes to the rank that owns its *anchor* (slot-0)
variable, and variables are split into contiguous id ranges balanced by
the number of edges anchored in them.  That gives point ranges for the SVM
chain (cut set: the bias ``b`` plus G-1 boundary weight copies), disk
ranges of the collision triangle for packing (balanced by edge count), and
time ranges for MPC.

``LocalGraph`` is a frozen-graph-shaped view of one rank's part (same
attribute names as ``FactorGraph``) so the device plan builder and the CPU
oracle consume it unchanged.
"""

from __future__ import annotations

import numpy as np

from ._pairwise import grouped_reduce


def _factor_first_edges(graph):
    if hasattr(graph, "_factor_edge0"):
        return graph._factor_edge0[:-1]
    return np.array([f.edge_range[0] for f in graph.factors], dtype=np.int64)


def locality_order(graph):
    """Variable order that keeps each factor's variables together.

    Hubs (degree > max(8, 4 x median degree), e.g. the SVM bias) are
    ignored; every other variable is keyed by the smallest non-hub
    variable id over its incident factors (one hop), ties by id.  SVM:
    w_i and xi_i interleave by point; packing and MPC keep id order.
    Returns (order, position-of-variable, hub mask, factor anchors)."""
    V = len(graph.var_offsets) - 1
    f_first = _factor_first_edges(graph)
    E = len(graph.edge_var)
    deg = np.bincount(graph.edge_var, minlength=V)
    hub = deg > max(8.0, 4.0 * float(np.median(deg)))
    ev = graph.edge_var
    ef = np.repeat(np.arange(len(f_first)), np.diff(np.append(f_first, E)))
    big = np.iinfo(np.int64).max
    cand = np.where(hub[ev], big, ev)
    fmin = np.full(len(f_first), big, dtype=np.int64)
    np.minimum.at(fmin, ef, cand)
    allmin = np.full(len(f_first), big, dtype=np.int64)
    np.minimum.at(allmin, ef, ev)
    fmin = np.where(fmin == big, allmin, fmin)
    key = np.full(V, big, dtype=np.int64)
    np.minimum.at(key, ev, fmin[ef])
    key = np.where(hub, np.arange(V), key)
    order = np.lexsort((np.arange(V), key))
    pos = np.empty(V, dtype=np.int64)
    pos[order] = np.arange(V)
    # anchor: the non-hub slot variable earliest in the order
    epos = np.where(hub[ev], big, pos[ev])
    amin = np.full(len(f_first), big, dtype=np.int64)
    np.minimum.at(amin, ef, epos)
    apos_all = np.full(len(f_first), big, dtype=np.int64)
    np.minimum.at(apos_all, ef, pos[ev])
    anchor_pos = np.where(amin == big, apos_all, amin)
    return order, pos, hub, anchor_pos


def factor_owner(graph, world):
    """Rank of every factor: variables are cut into `world` contiguous
    ranges of the locality order, balanced by the edges of the factors
    anchored in them; a factor goes to its anchor's rank."""
    V = len(graph.var_offsets) - 1
    f_first = _factor_first_edges(graph)
    arity = np.diff(np.append(f_first, len(graph.edge_var)))
    _order, _pos, _hub, anchor_pos = locality_order(graph)
    load = np.bincount(anchor_pos, weights=arity, minlength=V)
    cum = np.cumsum(load)
    total = cum[-1] if V else 0.0
    bounds = np.array([int(np.searchsorted(cum, total * r / world, side="left")) + 1
                       for r in range(1, world)], dtype=np.int64)
    owner = np.searchsorted(bounds, anchor_pos, side="right").astype(np.int64)
    # a factor on a single variable (SVM slack, MPC cost, radius) follows
    # the rank of that variable's other factors when they agree: it would
    # otherwise make the variable a cut variable for no load-balance gain
    E = len(graph.edge_var)
    ef = np.repeat(np.arange(len(f_first)), arity)
    ev = graph.edge_var
    multi = arity[ef] > 1
    big = np.iinfo(np.int64).max
    lo = np.full(V, big, dtype=np.int64)
    hi = np.full(V, -1, dtype=np.int64)
    np.minimum.at(lo, ev[multi], owner[ef[multi]])
    np.maximum.at(hi, ev[multi], owner[ef[multi]])
    single = np.nonzero(arity == 1)[0]
    sv = ev[f_first[single]]
    ok = lo[sv] == hi[sv]
    owner[single[ok]] = lo[sv[ok]]
    del E
    return owner


class LocalGraph:
    """One rank's factors and the variables they touch.

    Attributes mirror ``FactorGraph`` (``edge_var``, ``edge_offsets``,
    ``var_offsets``, ``zmap``, ``rho_flat``, ``z_weights``, ``blocks`` ...)
    in LOCAL numbering; ``global_var``, ``global_edge``, ``global_factor``
    map back.  ``z_weights`` are the GLOBAL weights of each variable.
    ``cut_index[k]`` is the canonical position of local z component k in
    the all-gathered cut vector (-1 when the variable is not cut).
    """

    def __init__(self, graph, owner, rank):
        self.rank = rank
        f_first = _factor_first_edges(graph)
        F = len(f_first)
        arity = np.diff(np.append(f_first, len(graph.edge_var)))
        mine = np.nonzero(owner == rank)[0]
        self.global_factor = mine
        edges = (np.repeat(f_first[mine], arity[mine])
                 + _ragged_arange(arity[mine]))
        self.global_edge = edges
        gvars = graph.edge_var[edges]
        self.global_var = np.unique(gvars)
        lv = np.searchsorted(self.global_var, gvars)
        dims_all = np.diff(graph.var_offsets)
        dims = dims_all[self.global_var]
        self.edge_var = lv.astype(np.int64)
        self.edge_rho = graph.edge_rho[edges].copy()
        self.edge_alpha = graph.edge_alpha[edges].copy()
        payload = dims[lv]
        self.edge_offsets = np.zeros(len(edges) + 1, dtype=np.int64)
        np.cumsum(payload, out=self.edge_offsets[1:])
        self.total_edge_payload = int(self.edge_offsets[-1])
        self.var_offsets = np.zeros(len(dims) + 1, dtype=np.int64)
        np.cumsum(dims, out=self.var_offsets[1:])
        self.z_dim = int(self.var_offsets[-1])
        self._zmap = self._rho_flat = self._alpha_flat = None   # built on first use
        # global payload positions of the local payload (for state scatter)
        gstart = graph.edge_offsets[edges]
        self.global_payload = np.repeat(gstart - self.edge_offsets[:-1], payload) + \
            np.arange(self.total_edge_payload)
        gz = graph.var_offsets[self.global_var]
        self.global_z = np.repeat(gz - self.var_offsets[:-1], dims) + np.arange(self.z_dim)
        self.z_weights = graph.z_weights[self.global_z].copy()
        # rho / alpha / z weights follow set_edge_params on the global
        # graph: re-sliced when its param_version moves (param_version)
        self._global = graph
        self._payload_len = payload
        self._version = getattr(graph, "param_version", None)
        # cut variables: local degree < global degree
        gdeg = np.bincount(graph.edge_var, minlength=len(dims_all))
        ldeg = np.bincount(lv, minlength=len(dims))
        self.var_cut = ldeg < gdeg[self.global_var]
        self._dims = dims
        # factor blocks restricted to this rank (creation order kept)
        self._blocks_local = []
        fe_local = np.zeros(len(mine) + 1, dtype=np.int64)
        np.cumsum(arity[mine], out=fe_local[1:])
        self._factor_edge0 = fe_local
        for cls, sdims, f0, vars_, params in graph.blocks:
            sel = np.nonzero((mine >= f0) & (mine < f0 + len(vars_)))[0]
            if sel.size == 0:
                continue
            rows = mine[sel] - f0
            lvars = np.searchsorted(self.global_var, vars_[rows])
            self._blocks_local.append((cls, sdims, int(sel[0]), lvars,
                                       _take_params(params, rows), sel))

    # ---- FactorGraph-compatible surface ------------------------------------
    @property
    def blocks(self):
        return [(c, d, f0, v, p) for c, d, f0, v, p, _s in self._blocks_local]

    def factor_first_edges(self, block_index):
        sel = self._blocks_local[block_index][5]
        return self._factor_edge0[sel]

    def _resync_params(self):
        g = self._global
        self.edge_rho = np.asarray(g.edge_rho)[self.global_edge].copy()
        self.edge_alpha = np.asarray(g.edge_alpha)[self.global_edge].copy()
        self._rho_flat = self._alpha_flat = None
        self.z_weights = np.asarray(g.z_weights)[self.global_z].copy()

    @property
    def zmap(self):
        if self._zmap is None:
            shift = self.var_offsets[self.edge_var] - self.edge_offsets[:-1]
            self._zmap = np.repeat(shift, self._payload_len) + np.arange(self.total_edge_payload)
        return self._zmap

    @property
    def rho_flat(self):
        self.param_version                      # re-slice after set_edge_params
        if self._rho_flat is None:
            self._rho_flat = np.repeat(self.edge_rho, self._payload_len)
        return self._rho_flat

    @property
    def alpha_flat(self):
        self.param_version
        if self._alpha_flat is None:
            self._alpha_flat = np.repeat(self.edge_alpha, self._payload_len)
        return self._alpha_flat

    @property
    def param_version(self):
        """The global graph's parameter version; the local rho, alpha and z
        weights are re-sliced from it whenever it moved (a graph without a
        version -- a reference FactorGraph -- is re-sliced on every read,
        and None makes the device plan re-sync every time)."""
        gv = getattr(self._global, "param_version", None)
        if gv is None or gv != self._version:
            self._resync_params()
            self._version = gv
        return gv

    def variable_slice(self, v):
        return slice(int(self.var_offsets[v]), int(self.var_offsets[v + 1]))

    def counts(self):
        return (len(self._dims), len(self.global_factor), len(self.edge_var))

    @property
    def edge_factor(self):
        return np.repeat(np.arange(len(self.global_factor)), np.diff(self._factor_edge0))


def _ragged_arange(lengths):
    lengths = np.asarray(lengths, dtype=np.int64)
    if lengths.size == 0:
        return np.zeros(0, dtype=np.int64)
    starts = np.repeat(np.cumsum(lengths) - lengths, lengths)
    return np.arange(int(lengths.sum()), dtype=np.int64) - starts


def _take_params(params, rows):
    out = {}
    for k, v in params.items():
        if k == "systems":
            out[k] = v
        elif isinstance(v, list):
            out[k] = [np.asarray(a)[rows] for a in v]
        else:
            out[k] = np.asarray(v)[rows]
    return out


class Partition:
    """A world-size split of one graph, identical on every rank."""

    def __init__(self, graph, world):
        self.world = int(world)
        self.owner = factor_owner(graph, self.world)
        self.locals = None
        self.graph = graph
        # canonical cut components: global z indices of cut variables, sorted
        gdeg = np.bincount(graph.edge_var, minlength=len(graph.var_offsets) - 1)
        edge_owner = np.repeat(self.owner, np.diff(np.append(_factor_first_edges(graph),
                                                             len(graph.edge_var))))
        V = len(graph.var_offsets) - 1
        first_owner = np.full(V, -1, dtype=np.int64)
        order = np.argsort(graph.edge_var, kind="stable")
        ev_sorted = graph.edge_var[order]
        starts = np.searchsorted(ev_sorted, np.arange(V))
        first_owner = edge_owner[order[starts]]
        differs = np.zeros(V, dtype=bool)
        np.logical_or.at(differs, ev_sorted, edge_owner[order] != first_owner[ev_sorted])
        self.var_cut = differs
        del gdeg
        dims = np.diff(graph.var_offsets)
        cut_vars = np.nonzero(differs)[0]
        self.cut_z = (np.repeat(graph.var_offsets[cut_vars], dims[cut_vars])
                      + _ragged_arange(dims[cut_vars]))
        self.ncut = len(self.cut_z)

    def local(self, rank):
        lg = LocalGraph(self.graph, self.owner, rank)
        lg.cut_index = np.full(lg.z_dim, -1, dtype=np.int64)
        pos = np.searchsorted(self.cut_z, lg.global_z)
        hit = (pos < self.ncut) & (self.cut_z[np.minimum(pos, max(self.ncut - 1, 0))]
                                   == lg.global_z) if self.ncut else np.zeros(lg.z_dim, bool)
        lg.cut_index[hit] = pos[hit]
        lg.ncut = self.ncut
        assert np.array_equal(lg.var_cut, self.var_cut[lg.global_var])
        return lg


def local_partial_sums(lg, m):
    """Per cut component of ``lg``: NumPy pairwise sum of m*rho over the
    local part of its segment (creation order); returns the canonical
    (ncut,) vector with zeros elsewhere (the rank's send buffer)."""
    vals = m * lg.rho_flat
    order = np.argsort(lg.zmap, kind="stable")
    ptr = np.searchsorted(lg.zmap[order], np.arange(lg.z_dim + 1))
    comps = np.nonzero(lg.cut_index >= 0)[0]
    sums = grouped_reduce(vals[order], ptr[comps], ptr[comps + 1] - ptr[comps])
    send = np.zeros(lg.ncut)
    send[lg.cut_index[comps]] = sums
    return send


def combine_partials(gathered):
    """Rank-order sum of all-gathered partials (G, ncut) -> (ncut,)."""
    out = np.array(gathered[0], dtype=np.float64, copy=True)
    for r in range(1, len(gathered)):
        out = out + gathered[r]
    return out


def local_weight_check(lg):
    """z_weights recomputed from local rho where the variable is not cut
    equal the global ones (same edges, same creation order)."""
    order = np.argsort(lg.edge_var, kind="stable")
    deg = np.bincount(lg.edge_var, minlength=len(lg.var_offsets) - 1)
    start = np.concatenate([[0], np.cumsum(deg)[:-1]])
    w = grouped_reduce(lg.edge_rho[order], start, deg)
    full = np.repeat(w, np.diff(lg.var_offsets))
    cut = np.repeat(lg.var_cut, np.diff(lg.var_offsets))
    return np.array_equal(full[~cut], lg.z_weights[~cut])


def svm_rank_graph(X, y, rank, world, lam=1.0, rho=1.0, alpha=1.0):
    """One rank's part of the SVM chain over the points of ALL ranks, built
    directly from this rank's points ``(X, y)`` (no global graph on the
    host: a weak-scaled run of world x n points fits where the global
    graph would not).

    It equals ``Partition(build_svm(...), world).local(rank)`` for the
    global SVM whose points are the ranks' blocks in rank order: the same
    local variables (this rank's w_i, the next rank's first weight copy as
    a cut variable with one equality edge, the bias, this rank's xi_i), the
    same factors in the same order, GLOBAL ``z_weights``, and the canonical
    cut vector ``[w of rank 1's first point (D), ..., w of rank G-1's
    (D), bias]``.  Every rank must hold the same number of points.
    """
    from .problems import SvmSpec, build_svm
    from ._pairwise import pairwise_sum
    X = np.asarray(X, dtype=np.float64)
    n, D = X.shape
    first, last = rank == 0, rank == world - 1
    N = n * world
    from .graph import GraphBuilder
    from .operators import Equality, SvmMargin, SvmNorm, SvmSlack
    spec = SvmSpec.from_arrays(X, y, lam=lam, rho=rho, alpha=alpha)
    Xs, ys = spec.arrays()
    b = GraphBuilder()
    w = b.declare_variables(D, n)
    wx = None if last else b.declare_variable(D)           # next rank's first w
    bias = b.declare_variable(1)
    xi = b.declare_variables(1, n)
    b.add_factors(SvmNorm, w[:, None], rho=rho, alpha=alpha,
                  params={"scale": np.full(n, 1.0 / N)}, slot_dims=(D,))
    b.add_factors(SvmSlack, xi[:, None], rho=rho, alpha=alpha,
                  params={"lam": np.full(n, float(lam))}, slot_dims=(1,))
    b.add_factors(SvmMargin, np.stack([w, np.full(n, bias), xi], axis=1), rho=rho,
                  alpha=alpha, params={"x": Xs, "y": ys}, slot_dims=(D, 1, 1))
    right = w[1:] if last else np.append(w[1:], wx)
    left = w[:-1] if last else w
    if len(left):
        b.add_factors(Equality, np.stack([left, right], axis=1), rho=rho, alpha=alpha,
                      slot_dims=(D, D))
    g = b.freeze()
    # global weights: sum of rho over the variable's incident edges of the
    # whole chain, in NumPy's pairwise order (graph.py:216-222)
    def wsum(deg):
        return float(pairwise_sum(np.full(deg, float(rho))))
    zw = np.array(g.z_weights, copy=True)
    dims = np.diff(np.asarray(g.var_offsets))
    def set_w(v, total):
        zw[g.var_offsets[v]:g.var_offsets[v] + dims[v]] = total
    w_end = wsum(3) if world * n > 1 else wsum(2)
    for i in range(n):
        deg = 4
        if first and i == 0:
            deg -= 1
        if last and i == n - 1:
            deg -= 1
        set_w(int(w[i]), wsum(deg))
    if wx is not None:
        set_w(int(wx), wsum(3 if rank + 1 == world - 1 and n == 1 else 4))
    set_w(int(bias), wsum(N))
    del w_end
    g.z_weights = zw
    # canonical cut vector positions
    cut = np.full(g.z_dim, -1, dtype=np.int64)
    ncut = (world - 1) * D + 1
    if world > 1:
        if not first:
            cut[g.var_offsets[int(w[0])]:g.var_offsets[int(w[0])] + D] = (rank - 1) * D + np.arange(D)
        if wx is not None:
            cut[g.var_offsets[int(wx)]:g.var_offsets[int(wx)] + D] = rank * D + np.arange(D)
        cut[g.var_offsets[int(bias)]] = (world - 1) * D
    g.cut_index = cut
    g.ncut = ncut if world > 1 else 0
    return g


def _mpc_owners(T, world):
    """Rank of every MPC factor under ``factor_owner``'s rule, from the
    horizon alone: anchors are nodes in id order (locality_order keeps id
    order: node t's key is t-1), a node's anchored load is cost (1 edge) +
    dyn_t (2 edges) + init (1 edge, node 0), and the single-variable
    factors follow their node's dynamics factors when those agree
    (cost_T follows dyn_{T-1}).  Returns (cost, dyn, init) owners."""
    load = np.full(T + 1, 3.0)
    load[T] = 1.0
    load[0] += 1.0
    cum = np.cumsum(load)
    total = cum[-1]
    bounds = np.array([int(np.searchsorted(cum, total * r / world, side="left")) + 1
                       for r in range(1, world)], dtype=np.int64)
    node_owner = np.searchsorted(bounds, np.arange(T + 1), side="right").astype(np.int64)
    dyn = node_owner[:T]
    cost = node_owner.copy()
    cost[T] = dyn[T - 1]                   # node T's only multi-variable factor
    return cost, dyn, int(node_owner[0])


def mpc_rank_graph(spec, rank, world):
    """One rank's part of ``build_mpc(spec)`` built from the spec alone (no
    global graph on the host).  Equals ``Partition(build_mpc(spec),
    world).local(rank)``: the same local variables (a contiguous node range,
    the boundary node of the next rank as a cut variable), the same factors
    in creation order, GLOBAL ``z_weights`` and the canonical cut vector
    (``tests/test_partition.py::test_mpc_rank_graph_equals_partition_local``)."""
    from .graph import GraphBuilder
    from .operators import MpcCost, MpcDyn, MpcInit
    from ._pairwise import pairwise_sum
    T = int(spec.horizon)
    d, k = spec.system.state_dim, spec.system.control_dim
    n0 = d + k
    cost_o, dyn_o, init_o = _mpc_owners(T, world)
    own_cost = np.nonzero(cost_o == rank)[0]
    own_dyn = np.nonzero(dyn_o == rank)[0]
    own_init = init_o == rank
    used = np.unique(np.concatenate([own_cost, own_dyn, own_dyn + 1,
                                     [0] if own_init else []]).astype(np.int64))
    if len(used) == 0:
        raise ValueError(f"rank {rank} of {world} owns no factor of a horizon-{T} MPC")
    lo = int(used[0])
    if not np.array_equal(used, np.arange(lo, lo + len(used))):
        raise AssertionError("MPC rank nodes are not contiguous")
    b = GraphBuilder()
    nodes = b.declare_variables(n0, len(used))          # local node t - lo
    diag = np.tile(np.concatenate([spec.q_diag, spec.r_diag]), (len(own_cost), 1))
    diag[own_cost == T, :d] = spec.qf_diag
    if len(own_cost):
        b.add_factors(MpcCost, nodes[own_cost - lo][:, None], rho=spec.rho, alpha=spec.alpha,
                      params={"diag": diag, "qdim": np.full(len(own_cost), d)},
                      slot_dims=(n0,))
    if len(own_dyn):
        b.add_factors(MpcDyn, np.stack([nodes[own_dyn - lo], nodes[own_dyn + 1 - lo]], axis=1),
                      rho=spec.rho, alpha=spec.alpha,
                      params={"systems": [spec.system],
                              "index": np.zeros(len(own_dyn), dtype=np.int64)},
                      slot_dims=(n0, n0))
    if own_init:
        b.add_factor(MpcInit(spec.q0, k), [int(nodes[0 - lo])], rho=spec.rho, alpha=spec.alpha)
    g = b.freeze()
    # global z weights: node t's incident edges in creation order are
    # [cost_t, dyn_{t-1} slot 1, dyn_t slot 0] (+ init at node 0; node T
    # has no dyn_T), summed in NumPy's pairwise order (graph.py:216-222)
    rho = float(spec.rho)
    deg = np.full(T + 1, 3)
    deg[T] = 2
    w = {int(n): float(pairwise_sum(np.full(n, rho))) for n in np.unique(deg)}
    zw = np.repeat(np.array([w[int(deg[t])] for t in used]), n0)
    g.z_weights = zw
    # cut nodes: incident factors on more than one rank
    cut_node = np.zeros(T + 1, dtype=bool)
    if world > 1:
        owners = [cost_o]
        prev = np.full(T + 1, -1)
        prev[1:] = dyn_o                    # dyn_{t-1} at node t
        nxt = np.full(T + 1, -1)
        nxt[:T] = dyn_o                     # dyn_t at node t
        init = np.full(T + 1, -1)
        init[0] = init_o
        allo = np.stack([cost_o, prev, nxt, init])
        valid = allo >= 0
        hi = np.where(valid, allo, -1).max(axis=0)
        lo_o = np.where(valid, allo, world).min(axis=0)
        cut_node = hi != lo_o
        del owners
    cut_nodes = np.nonzero(cut_node)[0]
    cut = np.full(g.z_dim, -1, dtype=np.int64)
    pos = {int(t): i for i, t in enumerate(cut_nodes)}
    for j, t in enumerate(used):
        if int(t) in pos:
            cut[j * n0:(j + 1) * n0] = pos[int(t)] * n0 + np.arange(n0)
    g.cut_index = cut
    g.ncut = len(cut_nodes) * n0
    return g


def _packing_owners(N, S):
    """Ranks-independent pieces of ``factor_owner`` for ``build_packing``:
    anchor positions are variable ids (locality_order keeps id order: every
    variable meets disk 0's center, so all keys tie), center i = 2i, radius
    i = 2i + 1; the anchored load of center i is 4 (N-1-i) collision edges
    + 2 S wall edges, of radius i its radius factor (1 edge)."""
    load = np.empty(2 * N)
    load[0::2] = 4.0 * (N - 1 - np.arange(N)) + 2.0 * S
    load[1::2] = 1.0
    return np.cumsum(load)


def packing_rank_graph(spec, rank, world):
    """One rank's part of ``build_packing(spec)`` built from the spec alone
    (no global graph on the host).  Equals ``Partition(build_packing(spec),
    world).local(rank)``: collision pairs (i, j > i) for the rank's anchor
    disks i in creation order, their walls and radius factors, the rank's
    variables in id order, GLOBAL ``z_weights`` and the canonical cut
    vector (``tests/test_partition.py::test_packing_rank_graph_equals_partition_local``)."""
    from .graph import GraphBuilder
    from .operators import Collision, Radius, Wall
    from ._pairwise import pairwise_sum
    N, S = int(spec.n), len(spec.planes)
    cum = _packing_owners(N, S)
    total = cum[-1]
    bounds = np.array([int(np.searchsorted(cum, total * r / world, side="left")) + 1
                       for r in range(1, world)], dtype=np.int64)
    pos_owner = np.searchsorted(bounds, np.arange(2 * N), side="right").astype(np.int64)
    c_own = pos_owner[0::2]                     # collisions (i, .) and walls of disk i
    # radius i follows disk i's multi-variable factors when they agree
    lo_o = np.minimum(np.where(np.arange(N) > 0, c_own[0], c_own), c_own)
    prev = np.concatenate([[c_own[0]], c_own[:-1]])
    hi_o = np.maximum(np.where(np.arange(N) > 0, prev, c_own), c_own)
    r_own = np.where(lo_o == hi_o, lo_o, pos_owner[1::2])
    coll = np.nonzero(c_own == rank)[0] if N > 1 else np.zeros(0, dtype=np.int64)
    coll = coll[coll < N - 1]
    walls = np.nonzero(c_own == rank)[0]
    rads = np.nonzero(r_own == rank)[0]
    # used variables (global ids): partners j > i of the collision anchors,
    # the anchors, wall disks, radius variables
    parts = [2 * walls, 2 * walls + 1, 2 * rads + 1]
    if len(coll):
        a = int(coll.min())
        parts += [2 * coll, 2 * coll + 1, np.arange(2 * (a + 1), 2 * N)]
    used = np.unique(np.concatenate(parts).astype(np.int64))
    if len(used) == 0:
        raise ValueError(f"rank {rank} of {world} owns no factor of a {N}-disk packing")
    lid = np.full(2 * N, -1, dtype=np.int64)
    lid[used] = np.arange(len(used))
    b = GraphBuilder()
    dims = np.where(used % 2 == 0, 2, 1)
    for dm in dims:                              # declaration order = global id order
        b.declare_variable(int(dm))
    if len(coll):
        ii = np.repeat(coll, N - 1 - coll)
        starts = np.repeat(np.cumsum(N - 1 - coll) - (N - 1 - coll), N - 1 - coll)
        jj = ii + 1 + (np.arange(len(ii)) - starts)
        b.add_factors(Collision, np.stack([lid[2 * ii], lid[2 * ii + 1], lid[2 * jj],
                                           lid[2 * jj + 1]], axis=1),
                      rho=spec.rho, alpha=spec.alpha, slot_dims=(2, 1, 2, 1))
    if len(rads):
        b.add_factors(Radius, lid[2 * rads + 1][:, None], rho=spec.rho_radius, alpha=spec.alpha,
                      params={"kappa": np.full(len(rads), float(spec.kappa))}, slot_dims=(1,))
    if len(walls):
        normals = np.stack([p.normal for p in spec.planes])
        points = np.stack([p.point for p in spec.planes])
        b.add_factors(Wall, np.stack([np.repeat(lid[2 * walls], S), np.repeat(lid[2 * walls + 1], S)],
                                     axis=1),
                      rho=spec.rho, alpha=spec.alpha,
                      params={"Q": np.tile(normals, (len(walls), 1)),
                              "V": np.tile(points, (len(walls), 1))},
                      slot_dims=(2, 1))
    g = b.freeze()
    # global z weights: a center's incident edges are N-1 collisions then S
    # walls; a radius's N-1 collisions, its radius factor, S walls
    # (creation order), summed in NumPy's pairwise order
    rho, rr = float(spec.rho), float(spec.rho_radius)
    wc = float(pairwise_sum(np.full(N - 1 + S, rho)))
    wr = float(pairwise_sum(np.concatenate([np.full(N - 1, rho), [rr], np.full(S, rho)])))
    g.z_weights = np.concatenate([np.full(2, wc) if v % 2 == 0 else [wr] for v in used])
    # cut variables: incident factors on more than one rank (owners are
    # monotone in the anchor position, so a center j's collision owners span
    # c_own[0] .. c_own[j-1] plus c_own[j])
    idx = np.arange(N)
    first = np.where(idx > 0, c_own[0], c_own)
    cut_c = (first != c_own) if N > 1 else np.zeros(N, dtype=bool)
    cut_r = cut_c | (r_own != c_own)
    cut_var = np.empty(2 * N, dtype=bool)
    cut_var[0::2] = cut_c
    cut_var[1::2] = cut_r
    zoff = np.zeros(2 * N + 1, dtype=np.int64)
    zoff[1:] = np.cumsum(np.tile([2, 1], N))
    cut_vars = np.nonzero(cut_var)[0]
    cpos = np.zeros(2 * N, dtype=np.int64)
    cpos[cut_vars] = np.cumsum(np.tile([2, 1], N)[cut_vars]) - np.tile([2, 1], N)[cut_vars]
    cut = np.full(g.z_dim, -1, dtype=np.int64)
    loff = np.asarray(g.var_offsets)
    for j, v in enumerate(used):
        if cut_var[v]:
            dm = 2 if v % 2 == 0 else 1
            cut[loff[j]:loff[j] + dm] = cpos[v] + np.arange(dm)
    g.cut_index = cut
    g.ncut = int(np.tile([2, 1], N)[cut_vars].sum())
    g.global_var = used                         # for packing_init on the rank graph
    del zoff
    return g
