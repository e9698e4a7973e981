"""Device standard-form builder and finishing kernels vs the reference (GPU).

SURVEY §8(f) rows 2-3.  Fixtures: tests/golden/stdform_*.npz, written by the
real reference (oracle/make_golden_stdform.py).  Bit-exact for every array
(the device builds the same CSR arrays, b, c and map; restrict / lift /
unscale use scipy's summation order); violation scalars to 1e-12 relative
(their dot products are fixed-order trees, the reference's are OpenBLAS).
Full-size BASELINE configs 1 and 3 are checked against the oracle.
"""

from __future__ import annotations

import time

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import stdform_port as SF
from oracle.pdhg_port import KktPoint, Model, violation_summary
from test_stdform import NAMES, G, assert_same, check_std, load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import paper_2603_03150_b200 as e

    return e


class Scaling:
    def __init__(self, r, c):
        self.row_scale, self.col_scale = r, c


def close(a, b, tol=1e-12):
    return abs(a - b) <= tol * max(1.0, abs(b))


@pytest.mark.parametrize("name", NAMES)
def test_device_stdform_matches_reference(eng, name):
    z, g = load(name)
    p, fmap = eng.to_standard_form(g)
    check_std(z, p, fmap)


@pytest.mark.parametrize("name", NAMES)
def test_device_finishing_matches_reference(eng, name):
    from paper_2603_03150_b200 import finish

    z, g = load(name)
    p, fmap = eng.to_standard_form(g)
    un = finish.unscale_point(Scaling(z["row_scale"], z["col_scale"]),
                              KktPoint(z["pt_xs"], z["pt_ys"], z["pt_zs"]))
    for a, k in ((un.x, "un_x"), (un.y, "un_y"), (un.z, "un_z")):
        assert_same(a, z[k])
    x, y, zz = finish.restrict_point(g, fmap, un)
    for a, k in ((x, "r_x"), (y, "r_y"), (zz, "r_z")):
        assert_same(a, z[k])
    lifted = finish.lift_point(g, p, fmap, x, y)
    for a, k in ((lifted.x, "lift_x"), (lifted.y, "lift_y"), (lifted.z, "lift_z")):
        assert_same(a, z[k])
    v = finish.evaluate_general_point(g, x, y)
    ref = z["viol"]
    assert v.primal_inf == ref[0] and v.dual_inf == ref[1]        # maxima of bit-exact residuals
    assert close(v.rel_gap, ref[2]) and close(v.max_violation, ref[3])
    assert bool(v.comp_negative) == bool(z["viol_comp_negative"])


def test_device_stdform_validation(eng):
    T = eng.types()
    z, g = load("rand_12x20_s1")
    g.A = g.A.copy()
    g.A.data[3] = np.nan
    with pytest.raises(T.InvalidModelError, match="matrix entries must be finite"):
        eng.to_standard_form(g)
    z, g = load("boxed")
    g.lower = g.lower.copy()
    g.lower[1] = 5.0
    with pytest.raises(T.InvalidModelError, match="variable 1 has lower bound"):
        eng.to_standard_form(g)
    z, g = load("lp2")
    g.senses = ["<=", "=="]
    with pytest.raises(T.InvalidModelError, match="unknown row sense"):
        eng.to_standard_form(g)


@pytest.mark.parametrize("which", ["config1", "config3"])
def test_full_size_configs_match_oracle(eng, which):
    from paper_2603_03150_b200.instances import config1_general, config3_general

    g = config1_general(1.0) if which == "config1" else config3_general(1.0)
    t = time.perf_counter()
    p, fmap = eng.to_standard_form(g)
    t_dev = time.perf_counter() - t
    t = time.perf_counter()
    q, qmap = SF.to_standard_form(g)
    t_cpu = time.perf_counter() - t
    print(f"{which}: std form {p.A.shape} nnz={p.A.nnz}: device {t_dev:.2f}s (incl. upload/"
          f"download), numpy oracle {t_cpu:.2f}s")
    A, B = sp.csr_matrix(p.A), q.A
    assert_same(A.indptr.astype(np.int64), B.indptr.astype(np.int64))
    assert_same(A.indices.astype(np.int64), B.indices.astype(np.int64))
    assert_same(A.data, B.data)
    assert_same(p.b, q.b)
    assert_same(p.c, q.c)
    for k in ("shifts", "pos_col", "neg_col", "slack_of_row", "slack_coef", "bound_var"):
        assert_same(np.asarray(getattr(fmap, k)), np.asarray(getattr(qmap, k)))
    assert fmap.obj_shift == qmap.obj_shift


def test_config1_pipeline_matches_oracle(eng):
    """BASELINE config 1 (small): device standard form -> device Ruiz -> GPU
    PDHG -> device finishing, against the oracle's pipeline step by step."""
    from oracle import pdhg_port as OP
    from oracle.ruiz_port import ruiz_equilibrate as ruiz_port
    from paper_2603_03150_b200 import finish
    from paper_2603_03150_b200.instances import config1_general

    T = eng.types()
    g = config1_general(0.01, seed=5)
    p, fmap = eng.to_standard_form(g)
    q, qmap = SF.to_standard_form(g)
    scaled, info = eng.ruiz_equilibrate(p)
    qs, qinfo = ruiz_port(q)
    assert_same(sp.csr_matrix(scaled.A).data, qs.A.data)
    assert_same(info.col_scale, qinfo.col_scale)
    pt, st = eng.run_pdhg(scaled, T.PdhgParams(eps_rel=1e-4))
    opt, ost = OP.run_pdhg(Model(qs.A, qs.b, qs.c), OP.PdhgParams(eps_rel=1e-4))
    assert st.status.value == ost.status.value == "Optimal"
    assert st.iterations == ost.iterations and st.restarts == ost.restarts
    obj, oobj = float(scaled.c @ pt.x), float(qs.c @ opt.x)
    assert abs(obj - oobj) <= 1e-6 * max(1.0, abs(oobj))
    un = finish.unscale_point(info, pt)
    x, y, _ = finish.restrict_point(g, fmap, un)
    v = finish.evaluate_general_point(g, x, y)
    oun = SF.unscale_point(qinfo.row_scale, qinfo.col_scale, opt)
    ox, oy, _ = SF.restrict_point(g, qmap, oun)
    ov = SF.evaluate_general_point(g, ox, oy)
    assert np.allclose(x, ox, rtol=1e-6, atol=1e-6)
    assert v.max_violation <= 10 * max(ov.max_violation, 1e-6)
    # general-model objective within 1e-6 relative of the oracle's
    assert abs(g.c @ x - g.c @ ox) <= 1e-6 * max(1.0, abs(g.c @ ox))


def test_device_copy_invalidated_when_host_matrix_changes(eng):
    """stdform.device_csr serves the resident device matrix only while p.A is
    the matrix it was built from (a reassigned p.A must not be read
    through stale device arrays)."""
    from paper_2603_03150_b200 import stdform

    _, g = load("lp1")
    p, _ = eng.to_standard_form(g)
    assert stdform.device_csr(p) is not None
    p.A = sp.csr_matrix(p.A, copy=True)        # same values, new host buffers
    assert stdform.device_csr(p) is None
    # the Ruiz pass then uploads the new host matrix and still matches the oracle
    import oracle

    S, info = eng.ruiz_equilibrate(p)
    S_o, info_o = oracle.ruiz_equilibrate(p)
    np.testing.assert_array_equal(info.row_scale, info_o.row_scale)
