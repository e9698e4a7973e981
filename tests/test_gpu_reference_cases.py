"""The reference's own PDHG test cases, restated against the GPU engine.

Each test mirrors one in /root/reference/pkg/tests/test_pdhg.py (cited by
line) with the same inputs and assertions; the models come from the golden
files (built from the reference's _desk.py fixtures by oracle/make_golden.py).
"""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import paper_2603_03150_b200 as eng

    return eng


class _P:
    def __init__(self, A, b, c):
        self.A = sp.csr_matrix(np.asarray(A, dtype=float)) if not sp.issparse(A) else sp.csr_matrix(A)
        self.b = np.asarray(b, dtype=float)
        self.c = np.asarray(c, dtype=float)


def _set(dev, name, values):
    import torch

    with torch.cuda.stream(dev.stream):
        dev.vec(name)[: len(values)].copy_(torch.as_tensor(np.asarray(values, float), device=dev.device))
    dev.stream.synchronize()


def _step(eng, dev, tau, sigma, omega=1.0, k=1, iter0=0, w0=0.0):
    fail = dev.run_period(k, iter0, tau / omega, sigma * omega, w0)
    assert fail < 0
    return dev.fetch(0, want_z=False)


def test_opnorm_scalar_and_diagonal(eng):
    """test_pdhg.py:27-34"""
    assert eng.estimate_opnorm(sp.csr_matrix([[3.0]])) == pytest.approx(3.0)
    lam = eng.estimate_opnorm(sp.diags([1.0, 2.0, 5.0]).tocsr())
    assert lam <= 5.0 + 1e-9 and 5.0 <= 1.05 * lam


def test_opnorm_row_vector(eng):
    """test_pdhg.py:36-38"""
    assert eng.estimate_opnorm(sp.csr_matrix([[1.0, 1.0]])) == pytest.approx(np.sqrt(2.0), rel=0.05)


@pytest.mark.parametrize("seed", range(5))
def test_opnorm_bracket_against_dense_svd(eng, seed):
    """test_pdhg.py:40-47"""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((6, 9))
    lam = eng.estimate_opnorm(sp.csr_matrix(A), seed=seed)
    true = np.linalg.svd(A, compute_uv=False)[0]
    assert lam <= true + 1e-9
    assert true <= 1.05 * lam


def test_zero_matrix_rejected(eng):
    """test_pdhg.py:49-53"""
    T = eng.types()
    with pytest.raises(T.InvalidModelError):
        eng.estimate_opnorm(sp.csr_matrix((2, 2)))


def test_first_step_from_zero_lp1(eng):
    """test_pdhg.py:63-72: x+ = max(0, -tau c) = 0 and y+ = sigma b > 0."""
    gm = load_golden("lp1_std")
    norm = eng.estimate_opnorm(gm.A)
    dev = eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions())
    dev.reset()
    x, y, _ = _step(eng, dev, 0.5 / norm, 0.5 / norm)
    np.testing.assert_array_equal(x, [0.0, 0.0])
    np.testing.assert_allclose(y, [0.5 / norm * 1.0])
    assert y[0] > 0


def test_saddle_point_is_fixed(eng):
    """test_pdhg.py:74-81"""
    gm = load_golden("lp1_std")
    lam = eng.estimate_opnorm(gm.A)
    step = 1.0 / (1.05 * lam)
    dev = eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions())
    dev.reset()
    _set(dev, "x", [1.0, 0.0])
    _set(dev, "y", [1.0])
    x, y, _ = _step(eng, dev, step, step)
    np.testing.assert_allclose(x, [1.0, 0.0], atol=1e-15)
    np.testing.assert_allclose(y, [1.0], atol=1e-15)


def test_negative_entries_clamped(eng):
    """test_pdhg.py:83-88"""
    p = _P([[1.0]], [1.0], [100.0])
    lam = eng.estimate_opnorm(p.A)
    step = 1.0 / (1.05 * lam)
    dev = eng.DeviceLp(p.A, p.b, p.c, eng.GpuOptions())
    dev.reset()
    _set(dev, "x", [0.5])
    x, _, _ = _step(eng, dev, step, step)
    assert x[0] == 0.0


def test_projection_invariant_along_run(eng):
    """test_pdhg.py:90-96: x >= 0 after every one of 500 steps."""
    gm = load_golden("eq_10x18_s7_ruiz")
    lam = eng.estimate_opnorm(gm.A)
    step = 1.0 / (1.05 * lam)
    dev = eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions())
    dev.reset()
    for k in range(500):
        x, _, _ = _step(eng, dev, step, step, iter0=k, w0=float(k))
        assert np.all(x >= 0.0)


def test_merit_nonincreasing_in_saddle_metric(eng):
    """test_pdhg.py:98-120 on LP1: the step-scaled saddle metric never
    increases by more than 1e-9 per step over 2,000 steps."""
    gm = load_golden("lp1_std")
    xs, ys = np.array([1.0, 0.0]), np.array([1.0])
    lam = eng.estimate_opnorm(gm.A)
    tau = sigma = 1.0 / (1.05 * lam)
    A = gm.A.toarray()
    dev = eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions())
    dev.reset()

    def merit(x, y):
        dx, dy = x - xs, y - ys
        return dx @ dx / tau + dy @ dy / sigma + 2.0 * dy @ (A @ dx)

    prev = merit(np.zeros(2), np.zeros(1))
    for k in range(2000):
        x, y, _ = _step(eng, dev, tau, sigma, iter0=k, w0=float(k))
        cur = merit(x, y)
        assert cur <= prev + 1e-9
        prev = cur


def test_extract_reduced_costs_lp1(eng):
    """test_pdhg.py:124-132: z(y=1) = [0, 1]; z(0) = max(c, 0)."""
    gm = load_golden("lp1_std")
    dev = eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions())
    dev.reset()
    _, _, z = dev.fetch(0)
    np.testing.assert_array_equal(z, np.maximum(gm.c, 0.0))
    _set(dev, "y", [1.0])
    _, _, z = dev.fetch(0)
    np.testing.assert_array_equal(z, [0.0, 1.0])


def test_negative_part_becomes_dual_infeasibility(eng):
    """test_pdhg.py:134-142: c - A'y = -0.3 -> z = 0 and r_d = -0.3 (max|r_d| = 0.3)."""
    p = _P([[1.0]], [1.0], [0.7])
    dev = eng.DeviceLp(p.A, p.b, p.c, eng.GpuOptions())
    dev.reset()
    _set(dev, "y", [1.0])
    _, _, z = dev.fetch(0)
    assert z[0] == 0.0
    (q,) = dev.check(0)
    from paper_2603_03150_b200 import _native as N

    assert q[N.Q_RDMAX] == pytest.approx(0.3)


def test_lp1_converges_to_unique_optimum(eng):
    """test_pdhg.py:146-150"""
    gm = load_golden("lp1_std")
    T = eng.types()
    pt, st = eng.run_pdhg(gm, T.PdhgParams(eps_rel=1e-4))
    assert st.status.value == "Optimal"
    np.testing.assert_allclose(pt.x, [1.0, 0.0], atol=1e-3)


def test_tolerance_monotone_iterations(eng):
    """test_pdhg.py:162-169"""
    gm = load_golden("lp1_std")
    T = eng.types()
    its = {}
    for eps in (1e-4, 1e-8):
        _, st = eng.run_pdhg(gm, T.PdhgParams(eps_rel=eps))
        assert st.status.value == "Optimal"
        its[eps] = st.iterations
    assert its[1e-8] >= its[1e-4]


def test_iteration_limit(eng):
    """test_pdhg.py:195-200"""
    gm = load_golden("eq_10x18_s7_ruiz")
    T = eng.types()
    _, st = eng.run_pdhg(gm, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=128))
    assert st.status.value == "IterationLimit"
    assert st.iterations == 128


def test_restarts_happen(eng):
    """test_pdhg.py:202-210"""
    gm = load_golden("eq_20x35_s17_ruiz")
    T = eng.types()
    _, st = eng.run_pdhg(gm, T.PdhgParams(eps_rel=1e-6))
    assert st.status.value == "Optimal"
    assert st.restarts >= 1


def test_explicit_zero_matrix_raises_zero_division(eng):
    """stored explicit zeros pass the nnz guard, lam = 0 and
    the reference raises ZeroDivisionError at pdhg.py:119."""
    A = sp.csr_matrix((np.array([0.0, 0.0]), np.array([0, 1]), np.array([0, 1, 2])), shape=(2, 2))
    p = _P(A, [1.0, 1.0], [1.0, 1.0])
    with pytest.raises(ZeroDivisionError):
        eng.run_pdhg(p)
