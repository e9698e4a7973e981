"""Ruiz equilibration (transform.py:35-77): the oracle restatement pinned to
the reference outputs (CPU), and the device pass bit-identical to both (GPU)."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import GOLDEN, RUIZ_NAMES


class _P:
    def __init__(self, g):
        self.A = sp.csr_matrix((g["A_data"], g["A_indices"], g["A_indptr"]), shape=tuple(g["A_shape"]))
        self.b, self.c = g["b"].copy(), g["c"].copy()


def _canon(A):
    A = sp.csr_matrix(A, copy=True)
    A.sort_indices()
    return A


def _load(name):
    return np.load(GOLDEN / f"{name}.npz")


@pytest.mark.parametrize("name", RUIZ_NAMES)
def test_oracle_ruiz_matches_reference(name):
    import oracle

    g = _load(name)
    S, info = oracle.ruiz_equilibrate(_P(g))
    np.testing.assert_array_equal(info.row_scale, g["row_scale"])
    np.testing.assert_array_equal(info.col_scale, g["col_scale"])
    assert info.applied_iterations == int(g["applied"])
    ref = _canon(sp.csr_matrix((g["S_data"], g["S_indices"], g["S_indptr"]), shape=tuple(g["A_shape"])))
    got = _canon(S.A)
    np.testing.assert_array_equal(got.indptr, ref.indptr)
    np.testing.assert_array_equal(got.indices, ref.indices)
    np.testing.assert_array_equal(got.data, ref.data)
    np.testing.assert_array_equal(S.b, g["Sb"])
    np.testing.assert_array_equal(S.c, g["Sc"])


def test_empty_row_and_column_rejected_before_device_work():
    import paper_2603_03150_b200 as eng

    p = _P(_load(RUIZ_NAMES[0]))
    A = p.A.tolil()
    A[0, :] = 0
    p.A = sp.csr_matrix(A)
    p.A.eliminate_zeros()
    with pytest.raises(ValueError, match="row 0 has no nonzero entries"):
        eng.ruiz_equilibrate(p)


@pytest.mark.gpu
@pytest.mark.parametrize("name", RUIZ_NAMES)
def test_device_ruiz_bit_identical(name):
    import paper_2603_03150_b200 as eng

    g = _load(name)
    S, info = eng.ruiz_equilibrate(_P(g))
    np.testing.assert_array_equal(info.row_scale, g["row_scale"])
    np.testing.assert_array_equal(info.col_scale, g["col_scale"])
    assert info.applied_iterations == int(g["applied"])
    ref = _canon(sp.csr_matrix((g["S_data"], g["S_indices"], g["S_indptr"]), shape=tuple(g["A_shape"])))
    got = _canon(S.A)
    np.testing.assert_array_equal(got.indices, ref.indices)
    np.testing.assert_array_equal(got.data, ref.data)
    np.testing.assert_array_equal(S.b, g["Sb"])
    np.testing.assert_array_equal(S.c, g["Sc"])


@pytest.mark.gpu
def test_device_ruiz_then_pdhg_uses_device_layout():
    """The scaled matrix stays on the device: the following run_pdhg finds
    the registered layout (no second upload) and solves config 0 like the
    reference pipeline does (prepare_model -> run_pdhg)."""
    import paper_2603_03150_b200 as eng
    from conftest import load_golden

    g = _load("ruiz_config0")
    S, info = eng.ruiz_equilibrate(_P(g))
    lay = eng.device_lp(S, eng.GpuOptions())
    assert lay is eng.device_lp(S, eng.GpuOptions())
    T = eng.types()
    pt, st = eng.run_pdhg(S, T.PdhgParams(eps_rel=1e-4))
    ref = load_golden("config0_s0").run("e4")
    assert st.status.value == "Optimal"
    assert st.iterations == int(ref["iterations"])
    assert float(S.c @ pt.x) == pytest.approx(float(ref["obj"]), rel=1e-6)


@pytest.mark.gpu
def test_device_ruiz_scaled_config4():
    import oracle
    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.instances import config4

    p = config4(scale=0.01, seed=31)
    S, info = eng.ruiz_equilibrate(p, register_layout=False)
    So, io = oracle.ruiz_equilibrate(p)
    np.testing.assert_array_equal(info.row_scale, io.row_scale)
    np.testing.assert_array_equal(info.col_scale, io.col_scale)
    np.testing.assert_array_equal(_canon(S.A).data, _canon(So.A).data)


@pytest.mark.gpu
def test_empty_column_rejected():
    """transform.py:47-54: the first structurally empty column is named (checked on the device)."""
    import paper_2603_03150_b200 as eng

    p = _P(_load(RUIZ_NAMES[0]))
    A = p.A.tocsc()
    A[:, 3] = 0
    A = sp.csr_matrix(A)
    A.eliminate_zeros()
    p.A = A
    with pytest.raises(ValueError, match="column 3 has no nonzero entries"):
        eng.ruiz_equilibrate(p)


def _stored_zero_model():
    """A model whose A stores explicit zeros (MPS files can): 3 of them."""
    rng = np.random.default_rng(41)
    A = sp.random(30, 50, density=0.2, random_state=rng, format="csr")
    A.data = rng.standard_normal(A.nnz) * rng.uniform(0.1, 30.0, A.nnz)
    for r in range(30):                    # every row / column nonzero
        A[r, r] = 1.0 + r
    for j in range(30, 50):
        A[j - 30, j] = 2.0
    A = sp.csr_matrix(A)
    A.data[[0, 7, 19]] = 0.0               # stored zeros, not eliminated
    p = type("P", (), {})()
    p.A, p.b, p.c = A, rng.standard_normal(30), rng.standard_normal(50)
    return p


def test_oracle_ruiz_drops_stored_zeros_like_reference():
    """scipy's diags @ A @ diags drops stored zeros (transform.py:69): the
    restatement must do the same as the live reference (build container)."""
    import sys
    from pathlib import Path

    import oracle

    ref = Path("/root/reference/pkg/src")
    p = _stored_zero_model()
    S, info = oracle.ruiz_equilibrate(p)
    assert info.applied_iterations > 0
    assert S.A.nnz == p.A.nnz - 3 and np.all(S.A.data != 0.0)
    if not ref.exists():
        pytest.skip("reference tree not available (GPU box)")
    sys.path.insert(0, str(ref))
    try:
        import hybridlp

        R, rinfo = hybridlp.ruiz_equilibrate(hybridlp.StandardLp(p.A, p.b, p.c))
    finally:
        sys.path.remove(str(ref))
    np.testing.assert_array_equal(info.row_scale, rinfo.row_scale)
    got, want = _canon(S.A), _canon(R.A)
    np.testing.assert_array_equal(got.indptr, want.indptr)
    np.testing.assert_array_equal(got.indices, want.indices)
    np.testing.assert_array_equal(got.data, want.data)


@pytest.mark.gpu
def test_device_ruiz_drops_stored_zeros():
    """Device Ruiz on a matrix with stored zeros: structure, values and scales
    equal to the restatement (hence the reference), and PDHG runs on it."""
    import oracle
    import paper_2603_03150_b200 as eng

    p = _stored_zero_model()
    S_o, info_o = oracle.ruiz_equilibrate(p)
    S, info = eng.ruiz_equilibrate(p)
    np.testing.assert_array_equal(info.row_scale, info_o.row_scale)
    np.testing.assert_array_equal(info.col_scale, info_o.col_scale)
    got, want = _canon(S.A), _canon(S_o.A)
    assert got.nnz == want.nnz == p.A.nnz - 3
    np.testing.assert_array_equal(got.indptr, want.indptr)
    np.testing.assert_array_equal(got.indices, want.indices)
    np.testing.assert_array_equal(got.data, want.data)
    T = eng.types()
    pt, st = eng.run_pdhg(S, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=64))
    opt, ost = oracle.run_pdhg(S_o, oracle.PdhgParams(eps_rel=1e-12, max_kkt_passes=64))
    assert st.iterations == ost.iterations == 64
    np.testing.assert_allclose(pt.x, opt.x, rtol=0, atol=1e-9 * max(1.0, np.abs(opt.x).max()))
