"""Device Ruiz equilibration: drop-in for hybridlp.transform.ruiz_equilibrate.

transform.py:35-77 runs right before the PDHG path (prepare_model,
warmstart.py:178-197) and, on config 4, costs minutes on the CPU.  Here the
passes run on the GPU (csrc/ruiz.cu) with the reference's exact arithmetic,
so the scales and the scaled matrix are bit-identical to scipy's, and the
scaled matrix can stay on the device: the returned model's device layout is
registered in the engine's cache, so the following run_pdhg does not upload
it again.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _native as N
from . import hostio, streams


last_timings: dict = {}   # phase -> seconds of the latest ruiz_equilibrate call


class _ScalingError(ValueError):
    """Equilibration met a structurally empty row or column."""


@dataclass
class _ScalingInfo:
    row_scale: np.ndarray
    col_scale: np.ndarray
    applied_iterations: int


def _types():
    try:
        from hybridlp import lp_core, transform  # type: ignore

        return transform.ScalingError, transform.ScalingInfo, lp_core.StandardLp
    except ImportError:
        from .instances import Instance

        def make(A, b, c):
            return Instance("scaled", A, b, c)

        return _ScalingError, _ScalingInfo, make


def ruiz_equilibrate(p, max_iters: int = 20, tol: float = 1e-2, *, gpu=None, register_layout=True):
    """Iterative infinity-norm equilibration on the GPU (transform.py:35-77).

    Returns (scaled StandardLp, ScalingInfo), the reference's classes when
    hybridlp is importable.  Raises ScalingError on an empty row or column
    exactly like the reference (transform.py:47-54).
    """
    import torch

    from .engine import DeviceLp, GpuOptions, _as_csr, _cache_register

    ScalingError, ScalingInfo, StandardLp = _types()
    tm = {}
    t = time.perf_counter()
    A = _as_csr(p.A)
    m, n = A.shape
    row_nnz = np.diff(A.indptr)
    if (row_nnz == 0).any():
        i = int(np.nonzero(row_nnz == 0)[0][0])
        raise ScalingError(f"row {i} has no nonzero entries")
    if not torch.cuda.is_available():
        raise N.NativeError("ruiz_equilibrate needs a CUDA device; there is no CPU fallback")
    # the scaled matrix gets its own index arrays (as the reference's product
    # does): copied on a host thread while the device works
    idx_copy = hostio.submit(lambda: (A.indices.copy(), A.indptr.copy()))
    tm["host_checks_s"] = time.perf_counter() - t
    lib = N.load()
    opts = gpu or GpuOptions()
    dev = torch.device("cuda", torch.cuda.current_device() if opts.device is None else opts.device)
    with streams.Borrowed(dev) as stream, torch.cuda.device(dev), torch.cuda.stream(stream):
        from .stdform import device_csr

        t = time.perf_counter()
        resident = device_csr(p)   # built on this device by stdform.to_standard_form
        if resident is not None and resident[2].device == dev:
            ptr, col = resident[0], resident[1]
            val = resident[2].clone()    # scaled in place; the standard-form copy stays intact
        else:
            ptr, col, val = (hostio.h2d(A.indptr, np.int32, dev), hostio.h2d(A.indices, np.int32, dev),
                             hostio.h2d(A.data, np.float64, dev))
        # structurally empty columns (transform.py:47-54; rows were checked above)
        empty = torch.bincount(col[:A.nnz], minlength=n) == 0
        if bool(empty.any()):
            j = int(empty.nonzero()[0, 0])
            idx_copy.result()
            raise ScalingError(f"column {j} has no nonzero entries")
        rs = torch.empty(m, dtype=torch.float64, device=dev)
        cs = torch.empty(n, dtype=torch.float64, device=dev)
        tb = lib.pdhg_ruiz_tmp_bytes(m, n)
        tmp = torch.empty(tb, dtype=torch.uint8, device=dev)
        stream.synchronize()
        tm["upload_s"] = time.perf_counter() - t
        t = time.perf_counter()
        applied = C.c_int32()
        lo, hi = 1.0 / (1.0 + tol), 1.0 + tol                      # transform.py:59
        N.check(lib.pdhg_ruiz(m, n, int(A.nnz), ptr.data_ptr(), col.data_ptr(), val.data_ptr(),
                              rs.data_ptr(), cs.data_ptr(), int(max_iters), lo, hi,
                              tmp.data_ptr(), tb, stream.cuda_stream, C.byref(applied)))
        stream.synchronize()
        tm["passes_s"] = time.perf_counter() - t
        t = time.perf_counter()
        row_scale = hostio.d2h(rs)
        col_scale = hostio.d2h(cs)
        data = hostio.d2h(val)
    tm["download_s"] = time.perf_counter() - t
    t = time.perf_counter()
    indices, indptr = idx_copy.result()
    dropped = False
    if applied.value > 0 and not np.all(data != 0.0):
        # the reference rebuilds A as diags(r) @ A @ diags(c) (transform.py:69);
        # scipy's csr_matmat keeps only nonzero products, so stored zeros (and
        # products that underflow to zero) leave the structure.  Same here, in
        # row order; the device layout is then built from the compacted arrays.
        keep = data != 0.0
        counts = np.add.reduceat(keep.astype(np.int64), indptr[:-1]) if data.size else np.zeros(0, np.int64)
        counts[np.diff(indptr) == 0] = 0
        indptr = np.concatenate([[0], np.cumsum(counts)]).astype(indptr.dtype)
        data, indices = data[keep], indices[keep]
        dropped = True
    S = sp.csr_matrix((data, indices, indptr), shape=A.shape)
    b = row_scale * np.asarray(p.b, dtype=float)                    # transform.py:75
    c = col_scale * np.asarray(p.c, dtype=float)
    scaled = StandardLp(S, b, c)
    info = ScalingInfo(row_scale, col_scale, int(applied.value))
    tm["assemble_s"] = time.perf_counter() - t
    t = time.perf_counter()
    if register_layout:
        # its own pooled stream: the arrays' producer work is complete (the
        # downloads above synchronised the Ruiz stream), and the context drains
        # its stream before the arrays go back to the allocator
        lay = DeviceLp(scaled.A, scaled.b, scaled.c, opts,
                       device_arrays=None if dropped else (ptr, col, val))
        _cache_register(scaled, lay, opts)
        torch.cuda.synchronize(dev)
    tm["layout_s"] = time.perf_counter() - t
    last_timings.clear()
    last_timings.update(tm)
    return scaled, info
