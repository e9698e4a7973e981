"""Device finishing of the PDHG point.

Drop-ins for the functions that run right after ``run_pdhg`` in the
reference pipeline (``finish_point``, warmstart.py:209-224):

* ``unscale_point``          transform.py:87-93
* ``restrict_point``         lp_core.py:371-385
* ``lift_point``             lp_core.py:388-427
* ``violation_summary``      lp_core.py:468-485
* ``evaluate_general_point`` lp_core.py:488-492 (device standard form + lift + violation)
* ``finish_point``           warmstart.py:209-224 (presolve replay stays the reference's
                             ``postsolve``; everything around it runs here)
* ``mu_target``, ``center_toward_target``, ``centered_start``  warmstart.py:62-107 --
                             the hand-off of the PDHG point to the reference IPM

Each is a composition of sm_100a kernels (csrc/finish.cu) behind the C ABI:
sparse products in scipy's csr_matvec order, elementwise steps with the
reference's numpy / builtin semantics, so restrict / lift / unscale are
bit-identical to the reference and the violation scalars agree to rounding
(fixed-order dot products instead of OpenBLAS ddot).
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref

import numpy as np

from . import _native as N
from . import hostio, streams
from .lp_types import resolve

_lock = threading.Lock()
_models: dict[int, tuple] = {}


def _torch_dev(gpu):
    import torch

    from .engine import GpuOptions

    if not torch.cuda.is_available():
        raise N.NativeError("finishing needs a CUDA device; there is no CPU fallback")
    opts = gpu or GpuOptions()
    dev = torch.device("cuda", torch.cuda.current_device() if opts.device is None else opts.device)
    return torch, dev


class _DevCsr:
    """A CSR matrix on the device plus its transpose (device radix-sort
    transpose = scipy's tocsc arrays, so products over it follow scipy's
    A.T @ y order)."""

    def __init__(self, A, torch, dev, stream, arrays=None):
        from .engine import _as_csr

        lib = N.load()
        A = _as_csr(A)
        self.m, self.n = A.shape
        self.nnz = int(A.nnz)
        t = lambda a, dt: hostio.h2d(a, dt, dev)
        with torch.cuda.stream(stream):
            if arrays is not None:
                self.ptr, self.col, self.val = arrays
            else:
                self.ptr, self.col, self.val = (t(A.indptr, np.int32), t(A.indices, np.int32),
                                                t(A.data, np.float64))
            e = lambda k, dt: torch.empty(max(k, 1), dtype=dt, device=dev)
            self.tptr, self.tcol, self.tval = e(self.n + 1, torch.int32), e(self.nnz, torch.int32), \
                e(self.nnz, torch.float64)
            tb = lib.pdhg_transpose_tmp_bytes(self.nnz, self.m, self.n)
            tmp = torch.empty(max(tb, 1), dtype=torch.uint8, device=dev)
            N.check(lib.pdhg_transpose_csr(self.m, self.n, self.nnz, self.ptr.data_ptr(),
                                           self.col.data_ptr(), self.val.data_ptr(),
                                           self.tptr.data_ptr(), self.tcol.data_ptr(),
                                           self.tval.data_ptr(), tmp.data_ptr(), tb,
                                           stream.cuda_stream))
            stream.synchronize()

    def spmv(self, lib, transpose, v, base, out, stream):
        """out = A v | A' v (scipy order), or base - (...) when base is given."""
        rows = self.n if transpose else self.m
        p, c, a = (self.tptr, self.tcol, self.tval) if transpose else (self.ptr, self.col, self.val)
        N.check(lib.pdhg_spmv_seq(rows, p.data_ptr(), c.data_ptr(), a.data_ptr(), v.data_ptr(),
                                  base.data_ptr() if base is not None else None, out.data_ptr(),
                                  stream.cuda_stream))


def _dev_csr(model, torch, dev, stream) -> _DevCsr:
    """Device copy of ``model.A`` (cached per model object, weakly)."""
    from .stdform import device_csr

    A = model.A
    key = (id(model), dev.index)
    fp = (A.shape, int(A.nnz), A.data.ctypes.data if A.nnz else 0)
    with _lock:
        ent = _models.get(key)
    if ent is not None and ent[0]() is model and ent[1] == fp:
        return ent[2]
    resident = device_csr(model)
    arrays = resident if resident is not None and resident[2].device == dev else None
    d = _DevCsr(A, torch, dev, stream, arrays=arrays)
    try:
        ref = weakref.ref(model, lambda _r, k=key: _models.pop(k, None))
    except TypeError:
        return d
    with _lock:
        while len(_models) >= 8:
            _models.pop(next(iter(_models)))
        _models[key] = (ref, fp, d)
    return d


def _up(torch, dev, a, dt=np.float64):
    return hostio.h2d(a, dt, dev)


def unscale_point(s, pt_scaled, *, gpu=None):
    """transform.py:87-93: x = C x_s, y = R y_s, z = z_s / C (on the device)."""
    T = resolve()
    torch, dev = _torch_dev(gpu)
    lib = N.load()
    n, m = np.asarray(pt_scaled.x).size, np.asarray(pt_scaled.y).size
    with streams.Borrowed(dev) as stream, torch.cuda.device(dev), torch.cuda.stream(stream):
        rs, cs = _up(torch, dev, s.row_scale), _up(torch, dev, s.col_scale)
        xs, ys, zs = (_up(torch, dev, v) for v in (pt_scaled.x, pt_scaled.y, pt_scaled.z))
        x, y, z = (torch.empty(max(k, 1), dtype=torch.float64, device=dev) for k in (n, m, n))
        N.check(lib.pdhg_unscale_point(n, m, rs.data_ptr(), cs.data_ptr(), xs.data_ptr(), ys.data_ptr(),
                                       zs.data_ptr(), x.data_ptr(), y.data_ptr(), z.data_ptr(),
                                       stream.cuda_stream))
        out = (hostio.d2h(x[:n]), hostio.d2h(y[:m]), hostio.d2h(z[:n]))
    return T.KktPoint(*out)


def restrict_point(g, fmap, pt, *, gpu=None):
    """lp_core.py:371-385 on the device -> (x, y, z) over the general model."""
    T = resolve()
    if np.asarray(pt.x).size != fmap.n_std or np.asarray(pt.y).size != fmap.m_std:
        raise T.InvalidModelError("point does not match the standard form of this map")
    torch, dev = _torch_dev(gpu)
    lib = N.load()
    n, m = fmap.n_general, fmap.m_general
    with streams.Borrowed(dev) as stream, torch.cuda.device(dev), torch.cuda.stream(stream):
        G = _dev_csr(g, torch, dev, stream)
        xs = _up(torch, dev, pt.x)
        pos, neg = _up(torch, dev, fmap.pos_col, np.int32), _up(torch, dev, fmap.neg_col, np.int32)
        sh = _up(torch, dev, fmap.shifts)
        x = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        N.check(lib.pdhg_restrict_x(n, pos.data_ptr(), neg.data_ptr(), sh.data_ptr(), xs.data_ptr(),
                                    x.data_ptr(), stream.cuda_stream))
        y_h = np.asarray(pt.y, dtype=float)[:m].copy()
        y = _up(torch, dev, y_h if m else np.zeros(1))
        c = _up(torch, dev, g.c)
        z = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        G.spmv(lib, True, y, c, z, stream)                               # z = c - A'y
        out = (hostio.d2h(x[:n]), y_h, hostio.d2h(z[:n]))
    return out


def _lift_device(lib, torch, dev, stream, g, G, P, p, fmap, x, y):
    """lift_point on the device; returns device tensors (x_std, y_std, z_std)."""
    n, m = fmap.n_general, fmap.m_general
    ns, ms = fmap.n_std, fmap.m_std
    f = lambda k: torch.zeros(max(k, 1), dtype=torch.float64, device=dev)
    xd, yd = _up(torch, dev, x if n else np.zeros(1)), _up(torch, dev, y if m else np.zeros(1))
    pos, neg = _up(torch, dev, fmap.pos_col, np.int32), _up(torch, dev, fmap.neg_col, np.int32)
    x_std = f(ns)
    N.check(lib.pdhg_lift_x(n, xd.data_ptr(), _up(torch, dev, fmap.shifts).data_ptr(), pos.data_ptr(),
                            neg.data_ptr(), x_std.data_ptr(), stream.cuda_stream))
    b = _up(torch, dev, p.b)
    r = f(ms)
    P.spmv(lib, False, x_std, b, r, stream)                              # r = b - A x_std
    sl = _up(torch, dev, fmap.slack_of_row, np.int32)
    N.check(lib.pdhg_lift_slacks(ms, sl.data_ptr(), _up(torch, dev, fmap.slack_coef).data_ptr(),
                                 r.data_ptr(), x_std.data_ptr(), stream.cuda_stream))
    y_std = f(ms)
    if m:
        y_std[:m].copy_(yd[:m])
    bv = _up(torch, dev, fmap.bound_var, np.int32)
    if bool((np.asarray(fmap.bound_var) >= 0).any()):
        zg = f(n)
        G.spmv(lib, True, yd, _up(torch, dev, g.c), zg, stream)         # z_gen = c - A'y
        N.check(lib.pdhg_lift_bound_duals(ms, bv.data_ptr(), zg.data_ptr(), y_std.data_ptr(),
                                          stream.cuda_stream))
    c_std = _up(torch, dev, p.c)
    t = f(ns)
    P.spmv(lib, True, y_std, c_std, t, stream)                           # c - at_y(y_std)
    z_std = f(ns)
    N.check(lib.pdhg_max0(ns, t.data_ptr(), z_std.data_ptr(), stream.cuda_stream))
    return x_std, y_std, z_std, b, c_std


def lift_point(g, p, fmap, x, y, *, gpu=None):
    """lp_core.py:388-427 on the device -> KktPoint in the standard space."""
    T = resolve()
    x = np.asarray(x, dtype=float).ravel()
    y = np.asarray(y, dtype=float).ravel()
    for v, k in ((x, fmap.n_general), (y, fmap.m_general)):
        if v.size != k:
            raise T.InvalidModelError(f"expected array of length {k}, got {v.size}")
    torch, dev = _torch_dev(gpu)
    lib = N.load()
    with streams.Borrowed(dev) as stream, torch.cuda.device(dev), torch.cuda.stream(stream):
        G, P = _dev_csr(g, torch, dev, stream), _dev_csr(p, torch, dev, stream)
        xs, ys, zs, _, _ = _lift_device(lib, torch, dev, stream, g, G, P, p, fmap, x, y)
        ns, ms = fmap.n_std, fmap.m_std
        out = (hostio.d2h(xs[:ns]), hostio.d2h(ys[:ms]), hostio.d2h(zs[:ns]))
    return T.KktPoint(*out)


def _violation(T, lib, stream, P, b, c, x, y, z):
    tb = lib.pdhg_violation_tmp_bytes(P.m, P.n)
    import torch

    tmp = torch.empty(tb, dtype=torch.uint8, device=x.device)
    out = (C.c_double * 5)()
    N.check(lib.pdhg_violation(P.m, P.n, P.ptr.data_ptr(), P.col.data_ptr(), P.val.data_ptr(),
                               P.tptr.data_ptr(), P.tcol.data_ptr(), P.tval.data_ptr(), b.data_ptr(),
                               c.data_ptr(), x.data_ptr(), y.data_ptr(), z.data_ptr(), tmp.data_ptr(),
                               tb, stream.cuda_stream, out))
    primal_inf, dual_inf, cx, by, xz = (float(v) for v in out)
    rel_gap = xz / (1.0 + abs(cx))                                       # lp_core.py:478
    return T.ViolationSummary(primal_inf=primal_inf, dual_inf=dual_inf, rel_gap=rel_gap,
                              max_violation=max(primal_inf, dual_inf, rel_gap),
                              comp_negative=xz < 0)


def violation_summary(p, pt, *, gpu=None):
    """lp_core.py:468-485 on the device (residuals lp_core.py:430-444)."""
    T = resolve()
    x, y, z = (np.asarray(v, dtype=float).ravel() for v in (pt.x, pt.y, pt.z))
    m, n = p.A.shape
    if x.size != n or y.size != m or z.size != n:
        raise T.InvalidModelError(
            f"point dims ({x.size}, {y.size}, {z.size}) do not match model ({n}, {m})")
    torch, dev = _torch_dev(gpu)
    lib = N.load()
    with streams.Borrowed(dev) as stream, torch.cuda.device(dev), torch.cuda.stream(stream):
        P = _dev_csr(p, torch, dev, stream)
        u = lambda v: _up(torch, dev, v if v.size else np.zeros(1))
        return _violation(T, lib, stream, P, u(np.asarray(p.b, dtype=float)),
                          u(np.asarray(p.c, dtype=float)), u(x), u(y), u(z))


def evaluate_general_point(g, x, y, *, gpu=None):
    """lp_core.py:488-492: the general point's violation on its standard form,
    all on the device (standard form built by csrc/stdform.cu)."""
    from .stdform import to_standard_form

    T = resolve()
    p, fmap = to_standard_form(g, gpu=gpu)
    x = np.asarray(x, dtype=float).ravel()
    y = np.asarray(y, dtype=float).ravel()
    for v, k in ((x, fmap.n_general), (y, fmap.m_general)):
        if v.size != k:
            raise T.InvalidModelError(f"expected array of length {k}, got {v.size}")
    torch, dev = _torch_dev(gpu)
    lib = N.load()
    with streams.Borrowed(dev) as stream, torch.cuda.device(dev), torch.cuda.stream(stream):
        G, P = _dev_csr(g, torch, dev, stream), _dev_csr(p, torch, dev, stream)
        xs, ys, zs, b, c = _lift_device(lib, torch, dev, stream, g, G, P, p, fmap, x, y)
        return _violation(T, lib, stream, P, b, c, xs, ys, zs)


def finish_point(prep, pt_solve, *, gpu=None):
    """warmstart.py:209-224: unscale, restrict, postsolve, measure.

    The presolve replay is the reference's own ``postsolve`` (host code,
    outside this path); unscale / restrict / both violation summaries run on
    the device.  Returns the reference's FinishedPoint."""
    from hybridlp import warmstart as W  # type: ignore
    from hybridlp.transform import postsolve  # type: ignore

    T = resolve()
    scaled_viol = None
    if prep.solve_model is not None:
        scaled_viol = violation_summary(prep.solve_model, pt_solve, gpu=gpu)
        pt_std = unscale_point(prep.scaling, pt_solve, gpu=gpu) if prep.scaling else pt_solve
        x_r, y_r, z_r = restrict_point(prep.reduced, prep.fmap, pt_std, gpu=gpu)
    else:
        x_r = np.zeros(prep.reduced.n_vars if prep.reduced is not None else 0)
        y_r = np.zeros(prep.reduced.n_rows if prep.reduced is not None else 0)
        z_r = np.zeros_like(x_r)
    restored = postsolve(prep.presolve_result.stack, T.KktPoint(x_r, y_r, z_r), prep.original)
    viol = evaluate_general_point(prep.original, restored.x, restored.y, gpu=gpu)
    return W.FinishedPoint(restored.x, restored.y, restored.z, viol, scaled_viol)


# ----------------------------------------------------------------- IPM hand-off


def mu_target(x, z, n: int, mu_min: float, *, gpu=None) -> float:
    """warmstart.py:62-68: max(x'z / n, mu_min), x'z on the device."""
    T = resolve()
    x = np.asarray(x, dtype=float)
    z = np.asarray(z, dtype=float)
    if x.size != n or z.size != n or n < 1:
        raise T.InvalidModelError("x and z must both have length n >= 1")
    torch, dev = _torch_dev(gpu)
    lib = N.load()
    with streams.Borrowed(dev) as stream, torch.cuda.device(dev), torch.cuda.stream(stream):
        a, b = _up(torch, dev, x.ravel()), _up(torch, dev, z.ravel())
        tb = lib.pdhg_dot_tmp_bytes()
        tmp = torch.empty(tb, dtype=torch.uint8, device=dev)
        out = C.c_double()
        N.check(lib.pdhg_dot(n, a.data_ptr(), b.data_ptr(), tmp.data_ptr(), tb, stream.cuda_stream,
                             C.byref(out)))
    return max(float(out.value) / n, mu_min)


def center_toward_target(x, z, mu: float, alpha_min: float, delta_max: float, *, gpu=None):
    """warmstart.py:71-96 on the device -> (x_new, z_new), bit-identical to the reference."""
    x = np.asarray(x, dtype=float).ravel()
    z = np.asarray(z, dtype=float).ravel()
    torch, dev = _torch_dev(gpu)
    lib = N.load()
    n = x.size
    with streams.Borrowed(dev) as stream, torch.cuda.device(dev), torch.cuda.stream(stream):
        xd, zd = _up(torch, dev, x if n else np.zeros(1)), _up(torch, dev, z if n else np.zeros(1))
        xo, zo = torch.empty_like(xd), torch.empty_like(zd)
        N.check(lib.pdhg_center_toward_target(n, xd.data_ptr(), zd.data_ptr(), float(mu), float(alpha_min),
                                              float(delta_max), xo.data_ptr(), zo.data_ptr(),
                                              stream.cuda_stream))
        return hostio.d2h(xo[:n]), hostio.d2h(zo[:n])


def centered_start(pt, params=None, *, gpu=None):
    """warmstart.py:99-107: perturb (x, z) toward max(x'z/n, mu_min); y untouched."""
    T = resolve()
    if params is None:
        try:
            from hybridlp.warmstart import WarmStartParams  # type: ignore

            params = WarmStartParams()
        except ImportError:
            from types import SimpleNamespace

            params = SimpleNamespace(mu_min=1e-6, alpha_min=1e-6, delta_max=1e-4)  # warmstart.py:47-52
    x = np.asarray(pt.x, dtype=float)
    mu = mu_target(x, pt.z, x.size, params.mu_min, gpu=gpu)
    xn, zn = center_toward_target(x, pt.z, mu, params.alpha_min, params.delta_max, gpu=gpu)
    return T.KktPoint(xn, np.asarray(pt.y, dtype=float).copy(), zn)
