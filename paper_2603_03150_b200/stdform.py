"""Device standard-form builder: drop-in for hybridlp.lp_core.to_standard_form.

lp_core.py:250-368 converts a GeneralLp to ``min c'x, Ax=b, x>=0`` with a
per-column Python loop and a COO -> CSR conversion -- seconds at config 1,
minutes at config 3/4 scale, and the step right before Ruiz and the PDHG
path (prepare_model, warmstart.py:178-197).  Here the
arrays are built on the GPU (csrc/stdform.cu), bit-identical to the
reference's, and the standard-form matrix stays on the device: the device
Ruiz pass (ruiz.py) picks it up without a second upload.
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref

import numpy as np
import scipy.sparse as sp

from . import _native as N
from . import hostio
from .lp_types import resolve

_SENSE_CODE = {"=": 0, "<=": 1, ">=": 2}   # PDHG_SENSE_* (lp_core.py:22-25)


class Dims(C.Structure):
    """struct pdhg_stdform_dims."""

    _fields_ = [("m_std", C.c_int32), ("n_std", C.c_int32), ("nnz_std", C.c_int64),
                ("n_struct", C.c_int32), ("n_ineq", C.c_int32), ("n_bound", C.c_int32),
                ("nonfinite_entries", C.c_int32)]


# device copies of standard-form matrices built here, keyed by id(StandardLp):
# (weakref to the model, (indptr, indices, data) torch tensors, device index)
_device_csr: dict[int, tuple] = {}
_lock = threading.Lock()


def _host_fingerprint(A):
    """What must still hold for the device arrays to describe ``p.A``: the same
    matrix object, shape, nnz and host buffers (a reassigned or resized p.A
    invalidates the device copy)."""
    try:
        return (id(A), tuple(A.shape), int(A.nnz), A.data.ctypes.data, A.indices.ctypes.data,
                A.indptr.ctypes.data)
    except AttributeError:
        return None


def device_csr(p):
    """(indptr, indices, data) device tensors of a model built by to_standard_form,
    or None (unknown model, or its host matrix changed since it was built)."""
    with _lock:
        ent = _device_csr.get(id(p))
    if ent is None or ent[0]() is not p:
        return None
    fp = _host_fingerprint(getattr(p, "A", None))
    if fp is None or fp != ent[2]:
        return None
    return ent[1]


def _register(p, arrays) -> None:
    key = id(p)
    try:
        ref = weakref.ref(p, lambda _r, k=key: _device_csr.pop(k, None))
    except TypeError:
        return
    fp = _host_fingerprint(getattr(p, "A", None))
    with _lock:
        _device_csr[key] = (ref, arrays, fp)


def _canonical_csr(A):
    """CSR with sorted column indices and no duplicates (what the reference's
    COO -> CSR conversion produces from any input)."""
    if not sp.isspmatrix_csr(A) and not isinstance(A, sp.csr_array):
        A = sp.csr_matrix(A, dtype=float)
    if A.dtype != np.float64:
        A = A.astype(np.float64)
    if not A.has_canonical_format:
        A = A.copy()
        A.sum_duplicates()
    return A


def _validate_host(T, g, c, rhs, lower, upper) -> None:
    """GeneralLp.validate (lp_core.py:74-90) up to the matrix check, which
    runs on the device (plan flag)."""
    if not np.all(np.isfinite(c)):
        raise T.InvalidModelError("objective coefficients must be finite")
    if not np.all(np.isfinite(rhs)):
        raise T.InvalidModelError("right-hand sides must be finite")


def _validate_rest(T, senses, lower, upper) -> None:
    bad = [s for s in senses if s not in _SENSE_CODE]
    if bad:
        raise T.InvalidModelError(f"unknown row sense {bad[0]!r}")
    crossed = np.nonzero(lower > upper)[0]
    if crossed.size:
        j = int(crossed[0])
        raise T.InvalidModelError(
            f"variable {j} has lower bound {lower[j]} above upper bound {upper[j]}")


def to_standard_form(g, *, gpu=None, register_device=True):
    """Convert a GeneralLp to pure standard form on the GPU (lp_core.py:250-368).

    Returns (StandardLp, StandardFormMap) -- the reference's classes when
    hybridlp is importable -- with arrays bit-identical to the reference's.
    Raises InvalidModelError with the reference's messages and check order
    (GeneralLp.validate, lp_core.py:74-90).
    """
    import torch

    from .engine import GpuOptions

    T = resolve()
    A = _canonical_csr(g.A)
    m, n = A.shape
    c = np.ascontiguousarray(g.c, dtype=np.float64)
    rhs = np.ascontiguousarray(g.rhs, dtype=np.float64)
    lower = np.ascontiguousarray(g.lower, dtype=np.float64)
    upper = np.ascontiguousarray(g.upper, dtype=np.float64)
    senses = list(g.senses)
    _validate_host(T, g, c, rhs, lower, upper)
    if A.nnz >= 2**31 - 1:
        raise ValueError("nnz >= 2^31 is not supported by the int32 layout")
    if not torch.cuda.is_available():
        raise N.NativeError("to_standard_form needs a CUDA device; there is no CPU fallback")
    lib = N.load()
    opts = gpu or GpuOptions()
    dev = torch.device("cuda", torch.cuda.current_device() if opts.device is None else opts.device)
    codes = np.fromiter((_SENSE_CODE.get(s, 3) for s in senses), dtype=np.int8, count=m)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.device(dev), torch.cuda.stream(stream):
        t = lambda a, dt: hostio.h2d(a, dt, dev)
        ptr, col, val = t(A.indptr, np.int32), t(A.indices, np.int32), t(A.data, np.float64)
        d_sense, d_lo, d_up = t(codes, np.int8), t(lower, np.float64), t(upper, np.float64)
        d_rhs, d_c = t(rhs, np.float64), t(c, np.float64)
        tb = lib.pdhg_stdform_tmp_bytes(m, n)
        tmp = torch.empty(max(tb, 1), dtype=torch.uint8, device=dev)
        dims = Dims()
        sp_ = stream.cuda_stream
        N.check(lib.pdhg_stdform_plan(m, n, int(A.nnz), ptr.data_ptr(), col.data_ptr(),
                                      val.data_ptr(), d_sense.data_ptr(), d_lo.data_ptr(),
                                      d_up.data_ptr(), tmp.data_ptr(), tb, sp_, C.byref(dims)))
        if dims.nonfinite_entries:
            raise T.InvalidModelError("matrix entries must be finite")
        _validate_rest(T, senses, lower, upper)
        ms, ns, nz = dims.m_std, dims.n_std, int(dims.nnz_std)
        i32, f64 = torch.int32, torch.float64
        e = lambda k, dt: torch.empty(max(k, 1), dtype=dt, device=dev)
        s_ptr, s_col, s_val = e(ms + 1, i32), e(nz, i32), e(nz, f64)
        b_std, c_std = e(ms, f64), e(ns, f64)
        shifts, pos_col, neg_col = e(n, f64), e(n, i32), e(n, i32)
        slack_of_row, slack_coef, bound_var = e(ms, i32), e(ms, f64), e(ms, i32)
        N.check(lib.pdhg_stdform_build(
            m, n, int(A.nnz), ptr.data_ptr(), col.data_ptr(), val.data_ptr(), d_sense.data_ptr(),
            d_rhs.data_ptr(), d_lo.data_ptr(), d_up.data_ptr(), d_c.data_ptr(), C.byref(dims),
            tmp.data_ptr(), tb, sp_, s_ptr.data_ptr(), s_col.data_ptr(), s_val.data_ptr(),
            b_std.data_ptr(), c_std.data_ptr(), shifts.data_ptr(), pos_col.data_ptr(),
            neg_col.data_ptr(), slack_of_row.data_ptr(), slack_coef.data_ptr(),
            bound_var.data_ptr()))
        h = lambda x, k: hostio.d2h(x[:k])
        A_std = sp.csr_matrix((h(s_val, nz), h(s_col, nz), h(s_ptr, ms + 1)), shape=(ms, ns))
        A_std.has_sorted_indices = True
        b_h, c_h = h(b_std, ms), h(c_std, ns)
        maps = [h(x, k) for x, k in ((shifts, n), (pos_col, n), (neg_col, n),
                                     (slack_of_row, ms), (slack_coef, ms), (bound_var, ms))]
    # obj_shift: obj_offset + sum_j c_j lo_j over finite, nonzero lo in column
    # order (lp_core.py:283), sequential like the reference's `+=`
    fin = np.isfinite(lower) & (lower != 0.0)
    terms = c[fin] * lower[fin]
    obj_shift = float(np.add.accumulate(np.concatenate(([float(getattr(g, "obj_offset", 0.0))],
                                                        terms)))[-1])
    p = T.StandardLp(A_std, b_h, c_h)
    fmap = T.StandardFormMap(
        n_general=n, m_general=m, n_std=ns, m_std=ms, obj_shift=obj_shift,
        shifts=maps[0], pos_col=maps[1].astype(np.int64), neg_col=maps[2].astype(np.int64),
        slack_of_row=maps[3].astype(np.int64), slack_coef=maps[4],
        bound_var=maps[5].astype(np.int64))
    if register_device and nz > 0:
        _register(p, (s_ptr[:ms + 1], s_col[:nz], s_val[:nz]))
    return p, fmap
