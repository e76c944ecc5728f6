"""Factor-graph construction with the reference's flat edge-ordered layout.

Same public API and the same arrays as ``fgadmm/graph.py`` (builder,
frozen graph, ``set_edge_params``, documents), built in bulk: factors are
held as *blocks* (one operator class, one slot signature, a (B, k)
variable matrix and stacked parameters) instead of one Python object per
factor and per edge, so the 12.5M-factor packing graph and the
multi-million-point SVM graphs of the benchmark can be frozen in seconds.
``factors``, ``edges`` and ``variables`` are lazy views that create the
reference's node objects on access.

Reference layout contract (``graph.py:171-222``): edges in factor creation
order, payload offsets by cumulative variable dims, ``zmap`` payload->z,
``rho_flat``/``alpha_flat`` repeated per payload entry, ``z_weights`` the
per-variable ``np.add.reduce`` of incident edge weights in creation order.
"""

from __future__ import annotations

import json
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np

from ._pairwise import grouped_reduce

DOCUMENT_VERSION = "fgadmm-v1"


@dataclass
class VariableNode:
    """One unknown block; ``degree``/``weight_sum`` filled at freeze."""

    id: int
    dim: int
    degree: int = 0
    weight_sum: float = 0.0


@dataclass
class FunctionNode:
    """One objective term applied to ``neighbor_vars``; ``edge_range`` is
    its half-open span of global edge ids."""

    id: int
    operator: object
    neighbor_vars: tuple
    edge_range: tuple = (0, 0)


@dataclass
class Edge:
    """Factor-variable incidence carrying rho and alpha."""

    factor: int
    var: int
    rho: float
    alpha: float
    payload_dim: int


def _edge_weights(value, count, name):
    arr = np.atleast_1d(np.asarray(value, dtype=float))
    if arr.size == 1:
        arr = np.full(count, float(arr[0]))
    if arr.shape != (count,):
        raise ValueError(
            f"{name} must be a scalar or one value per edge; "
            f"got {arr.size} values for {count} edges")
    if not np.all(arr > 0.0):
        raise ValueError(f"{name} must be positive")
    return arr


class _Block:
    """Consecutive factors sharing one operator class and slot signature."""

    __slots__ = ("cls", "dims", "vars", "rho", "alpha", "params", "instances")

    def __init__(self, cls, dims, vars_, rho, alpha, params, instances):
        self.cls = cls
        self.dims = tuple(int(d) for d in dims)
        self.vars = vars_          # (B, k) int64
        self.rho = rho             # (B, k) float64
        self.alpha = alpha
        self.params = params       # stack_params output
        self.instances = instances  # list of operators or None (bulk)

    @property
    def count(self):
        return self.vars.shape[0]

    def operator(self, i):
        if self.instances is not None:
            return self.instances[i]
        return self.cls.unstack(self.params, i, self.dims)


class GraphBuilder:
    """Accumulates variable and factor declarations before freezing."""

    def __init__(self):
        self._dims = []
        self._pending = []      # ("one", op, vars, rho, alpha) | ("block", _Block)
        self._nfactors = 0
        self._frozen = False

    def _check_open(self):
        if self._frozen:
            raise RuntimeError("builder is frozen; create a new GraphBuilder")

    def declare_variable(self, dim):
        """Register an unknown block of length ``dim``; returns its id."""
        self._check_open()
        dim = int(dim)
        if dim < 1:
            raise ValueError("variable dim must be >= 1")
        self._dims.append(dim)
        return len(self._dims) - 1

    def declare_variables(self, dim, count):
        """Bulk ``declare_variable``: ``count`` variables of one dim; ids."""
        self._check_open()
        dim, count = int(dim), int(count)
        if dim < 1:
            raise ValueError("variable dim must be >= 1")
        first = len(self._dims)
        self._dims.extend([dim] * count)
        return np.arange(first, first + count, dtype=np.int64)

    def add_factor(self, operator, variables, rho=1.0, alpha=1.0):
        """Attach ``operator`` to the listed variables; returns the factor id."""
        self._check_open()
        var_ids = [int(v) for v in variables]
        if not var_ids:
            raise ValueError("a factor needs at least one variable")
        if len(set(var_ids)) != len(var_ids):
            raise ValueError(f"duplicate variable in factor: {var_ids}")
        for v in var_ids:
            if not 0 <= v < len(self._dims):
                raise ValueError(f"unknown variable id {v}")
        dims = tuple(self._dims[v] for v in var_ids)
        sig = tuple(operator.slot_dims())
        if sig != dims:
            raise ValueError(
                f"operator '{operator.kind}' expects slot dims {sig}, "
                f"variables have dims {dims}")
        k = len(var_ids)
        rho = _edge_weights(rho, k, "rho")
        alpha = _edge_weights(alpha, k, "alpha")
        self._pending.append(("one", operator, var_ids, rho, alpha))
        self._nfactors += 1
        return self._nfactors - 1

    def add_factors(self, cls, variables, rho=1.0, alpha=1.0, params=None,
                    slot_dims=None):
        """Bulk ``add_factor``: B factors of one class in creation order.

        ``variables`` is a (B, k) id matrix; ``rho``/``alpha`` a scalar, a
        (k,) per-slot vector or a (B, k) matrix; ``params`` the class's
        ``stack_params`` dict for the B factors.  Returns the factor ids.
        """
        self._check_open()
        V = np.asarray(variables, dtype=np.int64)
        if V.ndim != 2 or V.shape[1] < 1:
            raise ValueError("variables must be a (B, k) id matrix")
        B, k = V.shape
        if B == 0:
            return np.empty(0, dtype=np.int64)
        nvars = len(self._dims)
        if V.min() < 0 or V.max() >= nvars:
            bad = V[(V < 0) | (V >= nvars)][0]
            raise ValueError(f"unknown variable id {int(bad)}")
        if k > 1:
            S = np.sort(V, axis=1)
            if np.any(S[:, 1:] == S[:, :-1]):
                raise ValueError("duplicate variable in factor")
        dims_arr = np.asarray(self._dims, dtype=np.int64)[V]
        if slot_dims is None:
            slot_dims = tuple(int(d) for d in dims_arr[0])
        if np.any(dims_arr != np.asarray(slot_dims)[None, :]):
            raise ValueError(
                f"operator '{cls.kind}' expects slot dims {tuple(slot_dims)}")
        rho = self._weights_matrix(rho, B, k, "rho")
        alpha = self._weights_matrix(alpha, B, k, "alpha")
        blk = _Block(cls, slot_dims, V, rho, alpha, params or {}, None)
        self._pending.append(("block", blk))
        first = self._nfactors
        self._nfactors += B
        return np.arange(first, first + B, dtype=np.int64)

    @staticmethod
    def _weights_matrix(value, B, k, name):
        arr = np.asarray(value, dtype=float)
        if arr.ndim == 0 or arr.size == 1:
            arr = np.full((B, k), float(arr.reshape(-1)[0]))
        elif arr.shape == (k,):
            arr = np.broadcast_to(arr, (B, k)).copy()
        elif arr.shape != (B, k):
            raise ValueError(f"{name} must be a scalar, (k,) or (B, k)")
        if not np.all(arr > 0.0):
            raise ValueError(f"{name} must be positive")
        return np.ascontiguousarray(arr)

    def _blocks(self):
        """Merge consecutive single factors of one class/signature."""
        blocks = []
        run = []

        def flush():
            if not run:
                return
            ops = [r[1] for r in run]
            cls = type(ops[0])
            blocks.append(_Block(
                cls, ops[0].slot_dims(),
                np.array([r[2] for r in run], dtype=np.int64),
                np.array([r[3] for r in run], dtype=float),
                np.array([r[4] for r in run], dtype=float),
                cls.stack_params(ops), ops))
            run.clear()

        for item in self._pending:
            if item[0] == "block":
                flush()
                blocks.append(item[1])
                continue
            op = item[1]
            if run and (type(run[0][1]) is not type(op)
                        or tuple(run[0][1].slot_dims()) != tuple(op.slot_dims())):
                flush()
            run.append(item)
        flush()
        return blocks

    def freeze(self):
        """Materialize the flat storage layout and return the graph."""
        self._check_open()
        if self._nfactors == 0:
            raise ValueError("graph has no factors")
        blocks = self._blocks()
        dims = np.asarray(self._dims, dtype=np.int64)
        deg = np.zeros(len(dims), dtype=np.int64)
        for b in blocks:
            deg += np.bincount(b.vars.ravel(), minlength=len(dims))
        orphans = np.nonzero(deg == 0)[0]
        if orphans.size:
            raise ValueError(f"variable {int(orphans[0])} has no incident factors")
        self._frozen = True
        return FactorGraph._from_blocks(dims, blocks)


class _Lazy(Sequence):
    """Read-only sequence materializing items on access."""

    def __init__(self, n, make):
        self._n = int(n)
        self._make = make

    def __len__(self):
        return self._n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._make(j) for j in range(*i.indices(self._n))]
        i = int(i)
        if i < 0:
            i += self._n
        if not 0 <= i < self._n:
            raise IndexError(i)
        return self._make(i)

    def __iter__(self):
        for j in range(self._n):
            yield self._make(j)


class FactorGraph:
    """Frozen bipartite graph with edge-ordered flat storage.

    Immutable except per-edge ``rho``/``alpha`` via ``set_edge_params``
    (which bumps ``param_version`` so device plans re-sync).
    """

    def __init__(self):
        raise TypeError("use GraphBuilder.freeze() or deserialize()")

    @classmethod
    def _from_blocks(cls, dims, blocks):
        self = object.__new__(cls)
        self._blocks = blocks
        self._var_dims = dims
        self.param_version = 0
        counts = [b.count for b in blocks]
        self._block_first = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        F = int(self._block_first[-1])

        # edges in factor creation order (graph.py:161-177)
        self.edge_var = np.concatenate([b.vars.ravel() for b in blocks]).astype(np.int64)
        arity = np.concatenate([np.full(b.count, b.vars.shape[1], dtype=np.int64)
                                for b in blocks])
        self._factor_edge0 = np.concatenate([[0], np.cumsum(arity)]).astype(np.int64)
        self.edge_factor = np.repeat(np.arange(F, dtype=np.int64), arity)
        self.edge_rho = np.concatenate([b.rho.ravel() for b in blocks]).astype(float)
        self.edge_alpha = np.concatenate([b.alpha.ravel() for b in blocks]).astype(float)

        payload = dims[self.edge_var]
        self.edge_offsets = np.zeros(len(self.edge_var) + 1, dtype=np.int64)
        np.cumsum(payload, out=self.edge_offsets[1:])
        self.total_edge_payload = int(self.edge_offsets[-1])
        self.var_offsets = np.zeros(len(dims) + 1, dtype=np.int64)
        np.cumsum(dims, out=self.var_offsets[1:])
        self.z_dim = int(self.var_offsets[-1])

        # zmap / rho_flat / alpha_flat (graph.py:189-204) are per payload
        # double: built on first use (the device plan never reads them), so a
        # large graph does not hold 3 x 8 bytes per payload double it does
        # not need
        self._zmap = self._rho_flat = self._alpha_flat = None

        # incidence in creation order and averaging weights (graph.py:206-222)
        self._incident_order = np.argsort(self.edge_var, kind="stable")
        self._degree = np.bincount(self.edge_var, minlength=len(dims)).astype(np.int64)
        self._incident_start = np.zeros(len(dims) + 1, dtype=np.int64)
        np.cumsum(self._degree, out=self._incident_start[1:])
        wsum = grouped_reduce(self.edge_rho[self._incident_order],
                              self._incident_start[:-1], self._degree)
        self._weight_sum = wsum
        self.z_weights = np.repeat(wsum, dims)
        self._incident_cache = None
        return self

    # ---- per-payload arrays, built on first use ----------------------------
    def _payload_len(self):
        return self._var_dims[self.edge_var]

    @property
    def zmap(self):
        """Payload position -> z position (graph.py:189-194), vectorized."""
        if self._zmap is None:
            shift = self.var_offsets[self.edge_var] - self.edge_offsets[:-1]
            self._zmap = np.repeat(shift, self._payload_len()) + np.arange(
                self.total_edge_payload, dtype=np.int64)
        return self._zmap

    @property
    def rho_flat(self):
        if self._rho_flat is None:
            self._rho_flat = np.repeat(self.edge_rho, self._payload_len())
        return self._rho_flat

    @property
    def alpha_flat(self):
        if self._alpha_flat is None:
            self._alpha_flat = np.repeat(self.edge_alpha, self._payload_len())
        return self._alpha_flat

    # ---- lazy reference views ---------------------------------------------
    @property
    def variables(self):
        return _Lazy(len(self._var_dims), lambda v: VariableNode(
            v, int(self._var_dims[v]), int(self._degree[v]),
            float(self._weight_sum[v])))

    def _factor_block(self, f):
        b = int(np.searchsorted(self._block_first, f, side="right") - 1)
        return b, f - int(self._block_first[b])

    def _make_factor(self, f):
        b, i = self._factor_block(f)
        blk = self._blocks[b]
        e0 = int(self._factor_edge0[f])
        return FunctionNode(f, blk.operator(i), tuple(int(v) for v in blk.vars[i]),
                            (e0, e0 + blk.vars.shape[1]))

    @property
    def factors(self):
        return _Lazy(int(self._block_first[-1]), self._make_factor)

    def _make_edge(self, e):
        v = int(self.edge_var[e])
        return Edge(int(self.edge_factor[e]), v, float(self.edge_rho[e]),
                    float(self.edge_alpha[e]), int(self._var_dims[v]))

    @property
    def edges(self):
        return _Lazy(len(self.edge_var), self._make_edge)

    @property
    def var_incident_edges(self):
        if self._incident_cache is None:
            self._incident_cache = np.split(self._incident_order,
                                            self._incident_start[1:-1])
        return self._incident_cache

    @property
    def blocks(self):
        """Factor blocks: (operator class, slot dims, first factor id,
        (B, k) variable ids, stacked params) in creation order."""
        return [(b.cls, b.dims, int(self._block_first[i]), b.vars, b.params)
                for i, b in enumerate(self._blocks)]

    def factor_first_edges(self, block_index):
        """First global edge id of every factor of one block."""
        lo = int(self._block_first[block_index])
        hi = int(self._block_first[block_index + 1])
        return self._factor_edge0[lo:hi]

    # ---- reference API ----------------------------------------------------
    def counts(self):
        """Return (variable count, factor count, edge count)."""
        return (len(self._var_dims), int(self._block_first[-1]), len(self.edge_var))

    def variable_slice(self, var_id):
        """Slice of ``z`` holding this variable."""
        return slice(int(self.var_offsets[var_id]), int(self.var_offsets[var_id + 1]))

    def _refresh_weight(self, var_id):
        lo, hi = self._incident_start[var_id], self._incident_start[var_id + 1]
        incident = self._incident_order[lo:hi]
        total = float(np.add.reduce(self.edge_rho[incident]))
        self._weight_sum[var_id] = total
        self.z_weights[self.var_offsets[var_id]:self.var_offsets[var_id + 1]] = total

    def set_edge_params(self, edge_id, rho, alpha):
        """Replace one edge's weights; not while a phase is in flight."""
        rho, alpha = float(rho), float(alpha)
        if rho <= 0.0 or alpha <= 0.0:
            raise ValueError("rho and alpha must be positive")
        e = int(edge_id)
        if not 0 <= e < len(self.edge_var):
            raise IndexError(edge_id)
        self.edge_rho[e] = rho
        self.edge_alpha[e] = alpha
        lo, hi = self.edge_offsets[e], self.edge_offsets[e + 1]
        if self._rho_flat is not None:
            self._rho_flat[lo:hi] = rho
        if self._alpha_flat is not None:
            self._alpha_flat[lo:hi] = alpha
        f = int(self.edge_factor[e])
        b, i = self._factor_block(f)
        j = e - int(self._factor_edge0[f])
        self._blocks[b].rho[i, j] = rho
        self._blocks[b].alpha[i, j] = alpha
        self._refresh_weight(int(self.edge_var[e]))
        self.param_version += 1

    def factor_values(self, z, factor_id):
        """Per-slot values of a factor's variables read from ``z``."""
        f = self.factors[factor_id]
        return [z[self.variable_slice(v)] for v in f.neighbor_vars]

    def objective_value(self, z):
        """Sum of factor objectives at the consensus values."""
        return float(sum(f.operator.objective(
            [z[self.variable_slice(v)] for v in f.neighbor_vars]) for f in self.factors))

    def constraint_violation(self, z):
        """Largest factor constraint violation at the consensus values."""
        return float(max(f.operator.violation(
            [z[self.variable_slice(v)] for v in f.neighbor_vars]) for f in self.factors))

    def serialize(self):
        """Render the graph as a versioned JSON document string."""
        doc = {
            "version": DOCUMENT_VERSION,
            "variables": [{"id": v, "dim": int(d)} for v, d in enumerate(self._var_dims)],
            "factors": [
                {
                    "operator": f.operator.kind,
                    "params": f.operator.to_params(),
                    "vars": list(f.neighbor_vars),
                    "rho": self.edge_rho[f.edge_range[0]:f.edge_range[1]].tolist(),
                    "alpha": self.edge_alpha[f.edge_range[0]:f.edge_range[1]].tolist(),
                }
                for f in self.factors
            ],
        }
        return json.dumps(doc, indent=1)


def serialize(graph):
    """Module-level alias for :meth:`FactorGraph.serialize`."""
    return graph.serialize()


def deserialize(document):
    """Rebuild a frozen graph from a document produced by ``serialize``.

    Raises ``ValueError`` on malformed documents and unknown kinds.
    """
    from .prox import operator_class
    from . import operators  # noqa: F401  (registry)

    if isinstance(document, (str, bytes)):
        try:
            document = json.loads(document)
        except json.JSONDecodeError as exc:
            raise ValueError(f"malformed graph document: {exc}") from exc
    if not isinstance(document, dict):
        raise ValueError("graph document must be a JSON object")
    version = document.get("version")
    if version != DOCUMENT_VERSION:
        raise ValueError(f"unsupported graph document version {version!r}; "
                         f"expected {DOCUMENT_VERSION!r}")
    for key in ("variables", "factors"):
        if key not in document:
            raise ValueError(f"graph document is missing the '{key}' list")
    builder = GraphBuilder()
    entries = document["variables"]
    for i, entry in enumerate(entries):
        if int(entry.get("id", -1)) != i:
            raise ValueError(f"variable ids must be contiguous from 0; entry {i} "
                             f"has id {entry.get('id')!r}")
        builder.declare_variable(int(entry["dim"]))
    for i, entry in enumerate(document["factors"]):
        for key in ("operator", "vars"):
            if key not in entry:
                raise ValueError(f"factor entry {i} is missing '{key}'")
        cls = operator_class(entry["operator"])
        var_ids = [int(v) for v in entry["vars"]]
        dims = []
        for v in var_ids:
            if not 0 <= v < len(entries):
                raise ValueError(f"factor entry {i} references unknown variable {v}")
            dims.append(int(entries[v]["dim"]))
        op = cls.from_params(entry.get("params", {}), dims)
        builder.add_factor(op, var_ids, rho=entry.get("rho", 1.0),
                           alpha=entry.get("alpha", 1.0))
    return builder.freeze()
