"""Generate tests/golden/stdform_*.npz from the REAL reference (TEST INFRASTRUCTURE).

Runs only in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_stdform.py

For each general LP it stores the inputs (A as CSR arrays, c, senses, rhs,
lower, upper, obj_offset) and the reference's to_standard_form output
(lp_core.py:250-368: A_std arrays, b, c and every StandardFormMap field),
plus one point through unscale_point / restrict_point / lift_point /
evaluate_general_point (transform.py:87-93, lp_core.py:371-427,488-492) for
the finishing functions.  Instances: the reference's
desk LPs (lp1, lp2, degenerate, free_var, boxed), random mixed-sense
models with shifted / free / boxed columns and explicit zeros, and small
BASELINE config 1 and config 3 models.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import scipy
import scipy.sparse as sp

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"

sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))
sys.path.insert(0, str(ROOT))

import hybridlp  # noqa: E402
from _desk import boxed_lp, degenerate_lp, free_var_lp, lp1, lp2  # noqa: E402

from paper_2603_03150_b200.instances import config1_general, config3_general  # noqa: E402


def random_general(seed: int, m: int, n: int, density: float = 0.3):
    """Mixed <=, >=, = rows; lower in {0, finite nonzero, -inf}; upper finite
    or inf; some explicit zeros; nonzero objective offset."""
    rng = np.random.default_rng(seed)
    mask = rng.random((m, n)) < density
    A = np.where(mask, rng.uniform(-2.0, 2.0, (m, n)), 0.0)
    for j in range(n):
        if not A[:, j].any():
            A[rng.integers(m), j] = 1.0
    S = sp.csr_matrix(A)
    z = rng.random(S.nnz) < 0.05                      # explicit zeros stay stored entries
    S.data[z] = 0.0
    senses = [rng.choice([hybridlp.LE, hybridlp.GE, hybridlp.EQ]) for _ in range(m)]
    kind = rng.random(n)
    lower = np.where(kind < 0.2, -np.inf, np.where(kind < 0.5, rng.uniform(-3, 3, n), 0.0))
    upper = np.where(rng.random(n) < 0.4, np.abs(lower) + rng.uniform(1, 5, n), np.inf)
    upper = np.where(np.isfinite(lower) | (rng.random(n) < 0.5), upper, np.inf)
    return hybridlp.GeneralLp(c=rng.standard_normal(n), A=S, senses=senses,
                              rhs=rng.standard_normal(m) * 3, lower=lower, upper=upper,
                              obj_offset=float(rng.standard_normal()))


def instances():
    out = {d.name: d.model for d in (lp1(), lp2(), degenerate_lp(), free_var_lp(), boxed_lp())}
    for s, (m, n) in enumerate(((5, 8), (12, 20), (30, 45), (60, 80))):
        out[f"rand_{m}x{n}_s{s}"] = random_general(100 + s, m, n)
    out["config1_s0.01"] = config1_general(0.01, seed=1).to_reference()
    out["config3_s0.002"] = config3_general(0.002, seed=3).to_reference()
    return out


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    for name, g in instances().items():
        p, fmap = hybridlp.to_standard_form(g)
        rng = np.random.default_rng(7)
        # a point in the scaled standard space -> unscale -> restrict -> lift / evaluate
        try:
            scaled, info = hybridlp.ruiz_equilibrate(p)
        except (hybridlp.transform.ScalingError, hybridlp.InvalidModelError):  # explicit zeros
            info = hybridlp.ScalingInfo(np.ones(p.m), np.ones(p.n), 0)
            scaled = p
        xs = np.abs(rng.standard_normal(p.n))
        ys = rng.standard_normal(p.m)
        zs = np.maximum(0.0, scaled.c - scaled.at_y(ys))
        pt_std = hybridlp.unscale_point(info, hybridlp.KktPoint(xs, ys, zs))
        xr, yr, zr = hybridlp.restrict_point(g, fmap, pt_std)
        lifted = hybridlp.lift_point(g, p, fmap, xr, yr)
        viol = hybridlp.evaluate_general_point(g, xr, yr)
        A = g.A
        np.savez_compressed(
            OUT / f"stdform_{name}.npz",
            numpy_version=np.__version__, scipy_version=scipy.__version__,
            g_data=A.data, g_indices=A.indices, g_indptr=A.indptr, g_shape=np.array(A.shape),
            g_c=g.c, g_senses=np.array(g.senses), g_rhs=g.rhs, g_lower=g.lower, g_upper=g.upper,
            g_obj_offset=g.obj_offset,
            s_data=p.A.data, s_indices=p.A.indices, s_indptr=p.A.indptr, s_shape=np.array(p.A.shape),
            s_b=p.b, s_c=p.c, obj_shift=fmap.obj_shift, shifts=fmap.shifts, pos_col=fmap.pos_col,
            neg_col=fmap.neg_col, slack_of_row=fmap.slack_of_row, slack_coef=fmap.slack_coef,
            bound_var=fmap.bound_var, n_std=fmap.n_std, m_std=fmap.m_std,
            row_scale=info.row_scale, col_scale=info.col_scale, pt_xs=xs, pt_ys=ys, pt_zs=zs,
            un_x=pt_std.x, un_y=pt_std.y, un_z=pt_std.z, r_x=xr, r_y=yr, r_z=zr,
            lift_x=lifted.x, lift_y=lifted.y, lift_z=lifted.z,
            viol=np.array([viol.primal_inf, viol.dual_inf, viol.rel_gap, viol.max_violation]),
            viol_comp_negative=viol.comp_negative,
        )
        print(name, p.A.shape, p.A.nnz)


if __name__ == "__main__":
    main()
