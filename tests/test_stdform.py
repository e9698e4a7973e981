"""Standard-form builder and finishing functions.

CPU: the oracle restatement (oracle/stdform_port.py) against the real
reference's outputs (tests/golden/stdform_*.npz, oracle/make_golden_stdform.py),
bit for bit.  GPU (marker gpu): the device builder (csrc/stdform.cu through
the C ABI) against the same fixtures, bit for bit, plus full-size configs 1
and 3 against the oracle.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import stdform_port as SF
from oracle.pdhg_port import InvalidModelError, KktPoint, violation_summary

GOLD = sorted((Path(__file__).parent / "golden").glob("stdform_*.npz"))
NAMES = [p.stem[len("stdform_"):] for p in GOLD]


class G:
    """GeneralLp stand-in rebuilt from a fixture."""

    def __init__(self, z):
        self.A = sp.csr_matrix((z["g_data"], z["g_indices"], z["g_indptr"]), shape=tuple(z["g_shape"]))
        self.c, self.rhs = z["g_c"], z["g_rhs"]
        self.lower, self.upper = z["g_lower"], z["g_upper"]
        self.senses = [str(s) for s in z["g_senses"]]
        self.obj_offset = float(z["g_obj_offset"])


def load(name):
    z = np.load(Path(__file__).parent / "golden" / f"stdform_{name}.npz")
    return z, G(z)


def assert_same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    assert a.tobytes() == b.astype(a.dtype).tobytes()


def check_std(z, p, fmap):
    A = sp.csr_matrix(p.A)
    assert A.shape == tuple(z["s_shape"])
    assert_same(np.asarray(A.indptr, np.int64), z["s_indptr"].astype(np.int64))
    assert_same(np.asarray(A.indices, np.int64), z["s_indices"].astype(np.int64))
    assert_same(A.data, z["s_data"])
    assert_same(p.b, z["s_b"])
    assert_same(p.c, z["s_c"])
    assert np.float64(fmap.obj_shift).tobytes() == np.float64(z["obj_shift"]).tobytes()
    for k in ("shifts", "slack_coef"):
        assert_same(getattr(fmap, k), z[k])
    for k in ("pos_col", "neg_col", "slack_of_row", "bound_var"):
        assert_same(np.asarray(getattr(fmap, k), np.int64), z[k].astype(np.int64))
    assert fmap.n_std == int(z["n_std"]) and fmap.m_std == int(z["m_std"])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_stdform_matches_reference(name):
    z, g = load(name)
    p, fmap = SF.to_standard_form(g)
    check_std(z, p, fmap)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_finishing_matches_reference(name):
    z, g = load(name)
    p, fmap = SF.to_standard_form(g)
    un = SF.unscale_point(z["row_scale"], z["col_scale"], KktPoint(z["pt_xs"], z["pt_ys"], z["pt_zs"]))
    for a, k in ((un.x, "un_x"), (un.y, "un_y"), (un.z, "un_z")):
        assert_same(a, z[k])
    x, y, zz = SF.restrict_point(g, fmap, un)
    for a, k in ((x, "r_x"), (y, "r_y"), (zz, "r_z")):
        assert_same(a, z[k])
    lifted = SF.lift_point(g, p, fmap, x, y)
    for a, k in ((lifted.x, "lift_x"), (lifted.y, "lift_y"), (lifted.z, "lift_z")):
        assert_same(a, z[k])
    v = SF.evaluate_general_point(g, x, y)
    got = np.array([v.primal_inf, v.dual_inf, v.rel_gap, v.max_violation])
    assert_same(got, z["viol"])
    assert bool(v.comp_negative) == bool(z["viol_comp_negative"])


def test_oracle_validation_messages():
    z, g = load("boxed")
    g.lower = g.lower.copy()
    g.lower[1] = 5.0
    with pytest.raises(InvalidModelError, match="variable 1 has lower bound"):
        SF.to_standard_form(g)
    z, g = load("lp2")
    g.senses = ["<=", "<>"]
    with pytest.raises(InvalidModelError, match="unknown row sense"):
        SF.to_standard_form(g)
    z, g = load("lp2")
    g.c = g.c.copy()
    g.c[0] = np.inf
    with pytest.raises(InvalidModelError, match="objective coefficients"):
        SF.to_standard_form(g)
