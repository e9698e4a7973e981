"""CPU test of the engine's host control flow (engine._run) against the oracle.

The device is replaced by a numpy test double that implements the C-ABI
semantics (run_period / check / restart / save_best / fetch) with exactly
the reference's numpy operations.  With that double, engine._run must
reproduce the oracle -- status, iterations, restarts, returned x/y/z and
termination sides -- bit for bit, including the best-point aliasing of the
running average and the failure exits.  This isolates control-flow bugs
from kernel rounding.  (The double is test-only; the product has no CPU path.)
"""

from __future__ import annotations

import time

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from conftest import GOLDEN_NAMES, load_golden
from oracle.pdhg_port import Model
from paper_2603_03150_b200 import _native as N
from paper_2603_03150_b200 import engine
from paper_2603_03150_b200.lp_types import resolve


class NumpyDevice:
    """Test double with the semantics of libpdhg_b200's context."""

    def __init__(self, A, b, c):
        self.A = sp.csr_matrix(A)
        self.At = self.A.tocsc()
        self.b, self.c = np.asarray(b, float), np.asarray(c, float)
        self.m, self.n = self.A.shape

    def at_y(self, y):
        return self.At.T @ y

    def opnorm(self, v0, tol=1e-4, max_iters=100):
        v = v0.copy()
        lam = 0.0
        for _ in range(max_iters):
            w = self.A.T @ (self.A @ v)
            nw = np.linalg.norm(w)
            if nw == 0.0:
                break
            new = np.sqrt(nw)
            v = w / nw
            if lam > 0 and abs(new - lam) <= tol * new:
                lam = new
                break
            lam = new
        w = self.A.T @ (self.A @ v)
        nw = np.linalg.norm(w)
        if nw > 0:
            lam = max(lam, float(np.sqrt(nw)))
        return float(lam)

    def reset(self):
        self.x = np.zeros(self.n)
        self.y = np.zeros(self.m)
        self.ax = np.zeros(self.n)
        self.ay = np.zeros(self.m)
        self.bx = np.zeros(self.n)
        self.by = np.zeros(self.m)
        self.bz = np.zeros(self.n)

    def run_period(self, iters, iter0, tau_w, sigma_w, w0):
        for j in range(iters):
            x_new = np.maximum(0.0, self.x - tau_w * (self.c - self.at_y(self.y)))
            y_new = self.y + sigma_w * (self.b - self.A @ (2.0 * x_new - self.x))
            self.x, self.y = x_new, y_new
            w = w0 + (j + 1)
            self.ax += (x_new - self.ax) / w
            self.ay += (y_new - self.ay) / w
            if not (np.all(np.isfinite(self.x)) and np.all(np.isfinite(self.y))):
                return iter0 + j + 1
        return -1

    def _xy(self, which):
        which &= 3
        if which == N.PT_AVG:
            return self.ax, self.ay
        if which == N.PT_BEST:
            return self.bx, self.by
        return self.x, self.y

    def check(self, *specs):
        out = []
        for s in specs:
            x, y = self._xy(s)
            z = self.bz if s & N.SPEC_BEST_Z else np.maximum(0.0, self.c - self.at_y(y))
            r_p = self.b - self.A @ x
            r_d = self.c - self.at_y(y) - z
            q = np.zeros(N.NQ)
            q[N.Q_RP2] = r_p.dot(r_p)
            q[N.Q_RPMAX] = np.max(np.abs(r_p))
            q[N.Q_BY] = float(self.b @ y)
            q[N.Q_RD2] = r_d.dot(r_d)
            q[N.Q_RDMAX] = np.max(np.abs(r_d))
            q[N.Q_CX] = float(self.c @ x)
            q[N.Q_XZ] = float(x @ z)
            out.append(q)
        return out

    def restart(self, which):
        if which == N.PT_CUR:
            self.ax, self.ay = self.x.copy(), self.y.copy()
        else:
            self.x, self.y = self.ax.copy(), self.ay.copy()

    def save_best(self, which, flags):
        x, y = self._xy(which)
        if flags & N.BEST_Z:
            self.bz = np.maximum(0.0, self.c - self.at_y(y))
        if flags & N.BEST_XY:
            self.bx, self.by = x.copy(), y.copy()

    def fetch(self, spec, want_z=True):
        x, y = self._xy(spec)
        z = None
        if want_z:
            z = self.bz.copy() if spec & N.SPEC_BEST_Z else np.maximum(0.0, self.c - self.at_y(y))
        return x.copy(), y.copy(), z


def run_host(p, params, seed=0):
    T = resolve()
    dev = NumpyDevice(p.A, p.b, p.c)
    return engine._run(T, dev, p, params, seed, engine.GpuOptions(), time.monotonic())


CASES = [("e4", 1e-4, 200_000), ("lim128", 1e-12, 128), ("lim200", 1e-12, 200), ("e6", 1e-6, 200_000)]


@pytest.mark.parametrize("name", GOLDEN_NAMES)
@pytest.mark.parametrize("tag,eps,limit", CASES)
def test_host_flow_bitwise_vs_oracle(name, tag, eps, limit):
    gm = load_golden(name)
    T = resolve()
    pt, st = run_host(gm, T.PdhgParams(eps_rel=eps, max_kkt_passes=limit))
    opt, ost = oracle.run_pdhg(Model(gm.A, gm.b, gm.c),
                               oracle.PdhgParams(eps_rel=eps, max_kkt_passes=limit))
    assert st.status.value == ost.status.value
    assert st.iterations == ost.iterations
    assert st.restarts == ost.restarts
    assert st.max_violation == ost.max_violation
    np.testing.assert_array_equal(pt.x, opt.x)
    np.testing.assert_array_equal(pt.y, opt.y)
    np.testing.assert_array_equal(pt.z, opt.z)
    for f in ("ok", "primal_lhs", "primal_rhs", "dual_lhs", "dual_rhs", "gap_lhs", "gap_rhs"):
        assert getattr(st.termination, f) == getattr(ost.termination, f), f
    assert len(st.history) == len(ost.history)
    # and the reference itself (golden) agrees
    r = gm.run(tag)
    assert st.iterations == int(r["iterations"])


def test_live_average_best_point_is_exercised():
    """At least one golden IterationLimit run returns a best point that kept
    following the running average after it was chosen (pdhg.py:147-148)."""
    hits = 0
    for name in GOLDEN_NAMES:
        gm = load_golden(name)
        for limit in (128, 200):
            p = Model(gm.A, gm.b, gm.c)
            holder = {}
            oracle.run_pdhg(p, oracle.PdhgParams(eps_rel=1e-12, max_kkt_passes=limit),
                            on_step=lambda st: holder.__setitem__("st", st))
            pt, _ = oracle.run_pdhg(p, oracle.PdhgParams(eps_rel=1e-12, max_kkt_passes=limit))
            st = holder["st"]
            if np.array_equal(pt.x, st.avg_x) and not np.array_equal(st.avg_x, st.x):
                hits += 1
    assert hits >= 1


def test_numerical_failure_path():
    """A step that overflows stops at that iteration (pdhg.py:194-196)."""
    A = sp.csr_matrix(np.array([[1.0, 1e300], [2.0, 1.0]]))
    p = Model(A, np.array([1.0, 1e308]), np.array([1e308, -1e308]))
    T = resolve()
    pt, st = run_host(p, T.PdhgParams(eps_rel=1e-6, max_kkt_passes=500))
    opt, ost = oracle.run_pdhg(p, oracle.PdhgParams(eps_rel=1e-6, max_kkt_passes=500))
    assert ost.status.value == "NumericalFailure"
    assert st.status.value == ost.status.value
    assert st.iterations == ost.iterations
    np.testing.assert_array_equal(pt.x, opt.x)


def test_time_limit_zero_host():
    gm = load_golden("lp2_ruiz")
    T = resolve()
    pt, st = run_host(gm, T.PdhgParams(time_limit_s=0.0))
    assert st.status.value == "TimeLimit" and st.iterations == 0
    assert pt.x.size == gm.n


def test_empty_model_raises():
    T = resolve()
    import paper_2603_03150_b200 as eng

    class P:
        pass

    p = P()
    p.A = sp.csr_matrix((0, 3))
    p.b, p.c = np.zeros(0), np.zeros(3)
    with pytest.raises(T.InvalidModelError):
        eng.run_pdhg(p)
    p.A = sp.csr_matrix((2, 2))
    p.b, p.c = np.zeros(2), np.zeros(2)
    with pytest.raises(T.InvalidModelError):
        eng.run_pdhg(p)


def test_params_validation_is_the_reference_class():
    T = resolve()
    with pytest.raises(ValueError):
        T.PdhgParams(eps_rel=0.0)
    with pytest.raises(ValueError):
        T.PdhgParams(restart_beta=1.0)
