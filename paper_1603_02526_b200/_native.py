"""ctypes binding of ``libfgadmm_b200.so`` (declared in include/fgadmm_b200.h).

The shared library is built in-tree (``build.py``); loading fails loudly
if it is missing: there is no host fallback for any operator or phase.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FGADMM_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("FGADMM_LIB") or os.path.join(_HERE, "libfgadmm_b200.so")

FG_MAX_SLOTS = 8
PHASE_IDS = {"x": 0, "m": 1, "z": 2, "u": 3, "n": 4}
PHASE_NAMES = ("x", "m", "z", "u", "n")
BUF_X, BUF_U0, BUF_U1, BUF_AUX, BUF_Z0, BUF_Z1 = 0, 1, 2, 3, 4, 5

ERR_INVALID, ERR_CUDA, ERR_UNSUPPORTED, ERR_NONFINITE = -1, -2, -3, -4

_p = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)


class GraphDesc(C.Structure):
    _fields_ = [("num_vars", C.c_int64), ("num_edges", C.c_int64),
                ("payload", C.c_int64), ("z_dim", C.c_int64),
                ("var_dim", _i32p), ("var_offsets", _i64p),
                ("edge_var", _i32p), ("edge_offsets", _i64p),
                ("chunk", C.c_int32), ("small_degree", C.c_int32),
                ("z_cut_index", _i32p), ("ncut", C.c_int64)]


class GroupDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nslots", C.c_int32),
                ("slot_dim", C.c_int32 * FG_MAX_SLOTS), ("count", C.c_int64),
                ("first_edge", _i64p), ("fparams", _dp), ("fstride", C.c_int32),
                ("tstride", C.c_int32), ("tables", _dp), ("ntables", C.c_int64),
                ("fsys", _i32p), ("iparam", C.c_int32), ("reserved", C.c_int32)]


class RunConfig(C.Structure):
    _fields_ = [("max_iterations", C.c_int64), ("primal_tol", C.c_double),
                ("dual_tol", C.c_double), ("first_reads_n", C.c_int32),
                ("timing", C.c_int32), ("graph_chunk", C.c_int32),
                ("reserved", C.c_int32)]


class RunResult(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int32),
                ("error_phase", C.c_int32), ("error_iteration", C.c_int64),
                ("primal", C.c_double), ("dual", C.c_double),
                ("ms_total", C.c_double), ("ms_edge_pass", C.c_double),
                ("ms_var_pass", C.c_double), ("ms_reduce", C.c_double),
                ("launches", C.c_int64)]


EXPORTS = {
    "fg_plan_create": (C.c_int, [C.POINTER(GraphDesc), C.POINTER(GroupDesc), C.c_int32,
                                 C.c_int32, C.POINTER(_p)]),
    "fg_plan_destroy": (None, [_p]),
    "fg_plan_info": (C.c_int, [_p, _i64p]),
    "fg_plan_forms": (C.c_int, [_p, C.POINTER(C.c_int32)]),
    "fg_plan_sync_params": (C.c_int, [_p, _dp, _dp, _dp]),
    "fg_state_upload": (C.c_int, [_p, _dp, _dp, _dp]),
    "fg_run": (C.c_int, [_p, C.POINTER(RunConfig), _dp, C.POINTER(RunResult)]),
    "fg_state_download": (C.c_int, [_p, _dp, _dp, _dp, _dp, _dp]),
    "fg_state_nonfinite": (C.c_int, [_p, _i64p]),
    "fg_run_phase_ms": (C.c_int, [_p, C.c_int64, _dp, _i64p]),
    "fg_debug_download": (C.c_int, [_p, C.c_int32, _dp]),
    "fg_profile_kernels": (C.c_int, [_p, C.c_int64, C.c_int32, C.c_char_p, _dp, _i64p,
                                     _i32p]),
    "fg_phase_upload": (C.c_int, [_p, _dp, _dp, _dp, _dp, _dp]),
    "fg_phase": (C.c_int, [_p, C.c_int32]),
    "fg_phase_download": (C.c_int, [_p, _dp, _dp, _dp, _dp, _dp]),
    "fg_residuals": (C.c_int, [_p, _dp, _dp, _dp, _dp, _dp]),
    "fg_evaluate": (C.c_int, [_p, _dp, _dp]),
    "fg_prox_eval": (C.c_int, [C.POINTER(GroupDesc), _dp, _dp, _dp, C.c_int32]),
    "fg_wproj": (C.c_int, [_dp, C.c_int32, C.c_int32, _dp, _dp, C.c_int64, _dp, C.c_int32]),
    "fg_selftest_div": (C.c_int, [_dp, _dp, C.c_int64, _dp, _dp, C.c_int32]),
    "fg_nccl_unique_id": (C.c_int, [C.c_char_p, C.c_char_p]),
    "fg_plan_attach_nccl": (C.c_int, [_p, C.c_char_p, C.c_char_p, C.c_int32, C.c_int32]),
    "fg_p2p_export": (C.c_int, [_p, C.c_int32, C.c_char_p]),
    "fg_plan_attach_p2p": (C.c_int, [_p, C.c_int32, C.c_int32, C.c_char_p, C.c_int64]),
    "fg_group_run": (C.c_int, [C.POINTER(_p), C.c_int32, C.POINTER(RunConfig), _dp,
                               C.POINTER(RunResult)]),
    "fg_host_alloc": (C.c_int, [C.c_int64, C.POINTER(_p)]),
    "fg_host_free": (C.c_int, [_p]),
    "fg_last_error": (C.c_char_p, []),
    "fg_abi_version": (C.c_int, []),
    "fg_device_count": (C.c_int, [_i32p]),
}

_lib = None


class NativeError(RuntimeError):
    """A failure reported by the C-ABI (CUDA error or unsupported input)."""


def load():
    """Load the in-tree engine library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python build.py` (or "
            f"__graft_entry__.build()) to compile the sm_100a engine; there is "
            f"no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc):
    if rc == 0:
        return
    msg = load().fg_last_error().decode(errors="replace")
    if rc == ERR_INVALID:
        raise ValueError(msg)
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise NativeError(msg)


def dptr(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def i32ptr(a):
    return a.ctypes.data_as(_i32p) if a is not None else None


def i64ptr(a):
    return a.ctypes.data_as(_i64p) if a is not None else None


def f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def device_count():
    n = C.c_int32(0)
    rc = load().fg_device_count(C.byref(n))
    return int(n.value) if rc == 0 else 0


def make_group_desc(kind_id, slot_dims, count, first_edge, dparams, keep):
    """Fill a GroupDesc; arrays it points at are appended to ``keep``."""
    g = GroupDesc()
    g.kind = int(kind_id)
    g.nslots = len(slot_dims)
    if g.nslots > FG_MAX_SLOTS:
        raise NotImplementedError(f"factors with more than {FG_MAX_SLOTS} slots")
    for j, d in enumerate(slot_dims):
        g.slot_dim[j] = int(d)
    g.count = int(count)
    fe = np.ascontiguousarray(first_edge, dtype=np.int64)
    keep.append(fe)
    g.first_edge = i64ptr(fe)
    if dparams.fparams is not None:
        fp = f64(dparams.fparams).reshape(count, -1) if count else f64(dparams.fparams)
        keep.append(fp)
        g.fparams = dptr(fp)
        g.fstride = int(fp.shape[1]) if fp.ndim == 2 else 0
    if dparams.tables is not None:
        tb = f64(dparams.tables)
        keep.append(tb)
        g.tables = dptr(tb)
        g.ntables = int(tb.shape[0])
        g.tstride = int(tb.shape[1])
    if dparams.fsys is not None:
        fs = np.ascontiguousarray(dparams.fsys, dtype=np.int32)
        keep.append(fs)
        g.fsys = i32ptr(fs)
    g.iparam = int(dparams.iparam)
    return g


def prox_eval(cls, params, dims, values, rhos, device=0):
    """Run one kind's prox kernel over a batch (ProxFactor.batch_eval)."""
    lib = load()
    B = int(values[0].shape[0])
    if B == 0:
        return [np.empty((0, d)) for d in dims]
    keep = []
    dp = cls.device_params(params, dims)
    g = make_group_desc(cls.device_kind, dims, B, np.arange(B, dtype=np.int64) * len(dims),
                        dp, keep)
    vals = np.ascontiguousarray(np.concatenate([v.reshape(-1) for v in values]))
    rh = np.ascontiguousarray(np.concatenate(rhos))
    out = np.empty_like(vals)
    check(lib.fg_prox_eval(C.byref(g), dptr(vals), dptr(rh), dptr(out), int(device)))
    res, off = [], 0
    for d in dims:
        res.append(out[off:off + B * d].reshape(B, d))
        off += B * d
    return res


def wproj(M, nv, w, device=0):
    """Weighted null-space projection of the rows of ``nv`` (operators.py:
    86-96) on the device (fg_wproj)."""
    lib = load()
    M = np.ascontiguousarray(M, dtype=np.float64)
    nv = np.ascontiguousarray(np.atleast_2d(nv), dtype=np.float64)
    w = np.ascontiguousarray(np.broadcast_to(np.atleast_2d(w), nv.shape), dtype=np.float64)
    out = np.empty_like(nv)
    r, D = M.shape
    rc = lib.fg_wproj(dptr(M), int(r), int(D), dptr(nv), dptr(w), int(nv.shape[0]),
                      dptr(out), int(device))
    if rc == ERR_NONFINITE:
        raise np.linalg.LinAlgError(load().fg_last_error().decode(errors="replace"))
    check(rc)
    return out


def selftest_div(x, y, device=0):
    """(engine inline division, runtime division) of x / y on the device."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    q, ref = np.empty_like(x), np.empty_like(x)
    check(load().fg_selftest_div(dptr(x), dptr(y), int(x.size), dptr(q), dptr(ref), int(device)))
    return q, ref


class _PinnedBlock:
    """Owner of one cudaHostAlloc block; freed when the last view dies."""

    def __init__(self, nbytes):
        self.ptr = C.c_void_p()
        check(load().fg_host_alloc(int(nbytes), C.byref(self.ptr)))
        self.nbytes = int(nbytes)

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value:
            try:
                load().fg_host_free(self.ptr)
            except Exception:
                pass
            self.ptr = None


def pinned_empty(shape, dtype=np.float64):
    """A numpy array in page-locked host memory (full-rate PCIe copies)."""
    dtype = np.dtype(dtype)
    n = int(np.prod(shape)) if np.ndim(shape) else int(shape)
    nbytes = max(1, n * dtype.itemsize)
    block = _PinnedBlock(nbytes)
    buf = (C.c_char * nbytes).from_address(block.ptr.value)
    arr = np.frombuffer(buf, dtype=dtype, count=n).reshape(shape)
    arr.flags.writeable = True
    buf._fg_block = block          # keep the allocation alive with the view
    return arr


