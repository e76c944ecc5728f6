"""Operator plugin contract and kind registry.

Mirrors the reference's plugin boundary (``fgadmm/prox.py:18-132``): a
factor operator has a registry ``kind``, per-slot dimensions, a host-side
parameter packer ``stack_params`` and a batched ``batch_eval``.  Here the
batched evaluation runs on the B200 through the C-ABI
(``fg_prox_eval``); there is no host numerics path.  Each kind also
declares how its stacked parameters map onto the device kernel's layout
(``device_params``).

``prox_reference`` (the reference's independent penalty minimizer) is
test infrastructure and lives with the oracle, not here.
"""

from __future__ import annotations

import numpy as np

_REGISTRY = {}


def register(cls):
    """Class decorator adding an operator to the name registry."""
    _REGISTRY[cls.kind] = cls
    return cls


def operator_class(kind):
    """Look up a registered operator class by its document name."""
    cls = _REGISTRY.get(kind)
    if cls is None:
        raise ValueError(f"unknown operator kind {kind!r}")
    return cls


def registered_kinds():
    """Sorted names of all registered operator kinds."""
    return sorted(_REGISTRY)


def check_prox_input(dims, values, rhos):
    """Validate one factor's prox input (reference ``prox.py:112-132``).

    Returns float 1-D arrays and float weights; raises ``ValueError`` on
    slot-count or dimension mismatches and on nonpositive weights.
    """
    if len(values) != len(dims) or len(rhos) != len(dims):
        raise ValueError(
            f"expected {len(dims)} slots, got {len(values)} values "
            f"and {len(rhos)} weights"
        )
    arrays = []
    for j, d in enumerate(dims):
        arr = np.atleast_1d(np.asarray(values[j], dtype=float))
        if arr.shape != (d,):
            raise ValueError(f"slot {j} expects dim {d}, got shape {arr.shape}")
        arrays.append(arr)
    weights = [float(r) for r in rhos]
    if any(not r > 0.0 for r in weights):
        raise ValueError("rho must be positive")
    return arrays, weights


class DeviceParams:
    """Per-group parameter block in the device kernel's layout.

    ``fparams``: (B, fstride) float64 per-factor rows; ``tables``:
    (ntables, tstride) shared rows indexed by ``fsys``; ``iparam``: one
    kind-specific integer.
    """

    __slots__ = ("fparams", "tables", "fsys", "iparam")

    def __init__(self, fparams=None, tables=None, fsys=None, iparam=0):
        self.fparams = fparams
        self.tables = tables
        self.fsys = fsys
        self.iparam = int(iparam)


class ProxFactor:
    """Base class for factor operators.

    Subclasses set ``kind`` and ``device_kind`` and implement
    ``slot_dims``; kinds with parameters implement ``stack_params``,
    ``device_params`` and ``unstack`` (rebuild one instance from stacked
    rows, used by graphs built in bulk).  ``eval`` wraps a batch of one so
    single and batched evaluation share the device kernel.
    """

    kind = None
    device_kind = None

    def slot_dims(self):
        raise NotImplementedError

    @classmethod
    def stack_params(cls, instances):
        return {}

    @classmethod
    def device_params(cls, params, slot_dims):
        return DeviceParams()

    @classmethod
    def unstack(cls, params, i, slot_dims):
        return cls()

    @classmethod
    def host_check(cls, params, rhos):
        """Validate a batch before launch; return (row, message) or None."""
        return None

    @classmethod
    def batch_eval(cls, params, values, rhos):
        """Evaluate a batch of factors of this kind on the GPU.

        ``values``: one ``(B, d_j)`` array per slot; ``rhos``: one
        ``(B,)`` array per slot; returns per-slot minimizers.
        """
        from . import _native

        values = [np.ascontiguousarray(np.asarray(v, dtype=np.float64))
                  for v in values]
        if values and values[0].ndim == 1:
            values = [v.reshape(-1, 1) for v in values]
        rhos = [np.ascontiguousarray(np.asarray(r, dtype=np.float64).reshape(-1))
                for r in rhos]
        dims = tuple(int(v.shape[1]) for v in values)
        bad = cls.host_check(params, rhos)
        if bad is not None:
            raise ValueError(bad[1])
        return _native.prox_eval(cls, params, dims, values, rhos)

    def eval(self, values, rhos):
        """Minimize ``f(s) + sum_j rho_j/2 ||s_j - n_j||^2`` for one factor."""
        dims = self.slot_dims()
        values, rhos = check_prox_input(dims, values, rhos)
        params = type(self).stack_params([self])
        out = type(self).batch_eval(
            params, [v.reshape(1, -1) for v in values],
            [np.array([r]) for r in rhos])
        return [o[0].copy() for o in out]

    def objective(self, values):
        return 0.0

    def violation(self, values):
        return 0.0

    def to_params(self):
        return {}

    @classmethod
    def from_params(cls, params, dims):
        return cls()
