"""numpy restatement of the reference's model transforms around the PDHG path
(TEST INFRASTRUCTURE, not product code).

* ``to_standard_form``        lp_core.py:250-368
* ``unscale_point``           transform.py:87-93   (§8(f) row 3)
* ``restrict_point``          lp_core.py:371-385
* ``lift_point``              lp_core.py:388-427
* ``evaluate_general_point``  lp_core.py:488-492

Vectorised where the reference loops in Python, keeping its arithmetic:
the bound shift of b is applied column by column in ascending column order
(lp_core.py:281-283) -- here as rounds over each row's k-th shifted entry,
which is the same sequence of roundings per row -- and obj_shift is the
same sequential sum (np.add.accumulate).  Pinned bit for bit to the real
reference by tests/test_stdform.py against tests/golden/stdform_*.npz
(oracle/make_golden_stdform.py).  Only tests/, smoke() and bench.py import it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .pdhg_port import InvalidModelError, KktPoint, Model, violation_summary

EQ, LE, GE = "=", "<=", ">="


@dataclass
class StandardFormMap:
    """lp_core.py:224-247."""

    n_general: int
    m_general: int
    n_std: int
    m_std: int
    obj_shift: float
    shifts: np.ndarray
    pos_col: np.ndarray
    neg_col: np.ndarray
    slack_of_row: np.ndarray
    slack_coef: np.ndarray
    bound_var: np.ndarray

    def slack_columns(self) -> np.ndarray:
        return self.slack_of_row[self.slack_of_row >= 0]


def validate(g) -> None:
    """GeneralLp.validate (lp_core.py:74-90), same order and messages."""
    if not np.all(np.isfinite(g.c)):
        raise InvalidModelError("objective coefficients must be finite")
    if not np.all(np.isfinite(g.rhs)):
        raise InvalidModelError("right-hand sides must be finite")
    if not np.all(np.isfinite(g.A.data)):
        raise InvalidModelError("matrix entries must be finite")
    bad = [s for s in g.senses if s not in (LE, GE, EQ)]
    if bad:
        raise InvalidModelError(f"unknown row sense {bad[0]!r}")
    crossed = np.nonzero(g.lower > g.upper)[0]
    if crossed.size:
        j = int(crossed[0])
        raise InvalidModelError(
            f"variable {j} has lower bound {g.lower[j]} above upper bound {g.upper[j]}")


def to_standard_form(g):
    """lp_core.py:250-368 -> (Model(A_std, b_std, c_std), StandardFormMap)."""
    validate(g)
    A = sp.csr_matrix(g.A, dtype=float)
    if not A.has_canonical_format:
        A = A.copy()
        A.sum_duplicates()                       # what the final COO -> CSR does
    m, n = A.shape
    lo = np.asarray(g.lower, dtype=float)
    up = np.asarray(g.upper, dtype=float)
    c = np.asarray(g.c, dtype=float)
    fin = np.isfinite(lo)                        # lp_core.py:277
    width = np.where(fin, 1, 2)
    pos_col = np.concatenate(([0], np.cumsum(width)[:-1])).astype(np.int64)
    neg_col = np.where(fin, -1, pos_col + 1).astype(np.int64)
    shifts = np.where(fin, lo, 0.0)
    n_struct = int(width.sum())
    senses = list(g.senses)
    ineq = np.array([s != EQ for s in senses], dtype=bool)
    coef_row = np.array([1.0 if s == LE else -1.0 if s == GE else 0.0 for s in senses])
    ineq_idx = np.cumsum(ineq) - ineq               # slack index per ineq row (lp_core.py:303-314)
    fub = np.isfinite(up)
    bound_j = np.nonzero(fub)[0]
    n_ineq, n_bound = int(ineq.sum()), int(bound_j.size)
    m_std, n_std = m + n_bound, n_struct + n_ineq + n_bound

    # structural entries of row i in input column order: (pos_col, a) [, (pos_col+1, -a)]
    rows_nnz = np.diff(A.indptr)
    r_of = np.repeat(np.arange(m), rows_nnz)
    j_of = A.indices.astype(np.int64)
    w_of = width[j_of]
    rlen = np.bincount(r_of, weights=w_of, minlength=m).astype(np.int64) + ineq
    blen = 2 + (~fin[bound_j]).astype(np.int64)
    s_ptr = np.concatenate(([0], np.cumsum(np.concatenate((rlen, blen))))).astype(np.int64)
    nnz = int(s_ptr[-1])
    s_col = np.empty(nnz, dtype=np.int64)
    s_val = np.empty(nnz)
    # position of each input entry inside its output row
    wcum = np.cumsum(w_of) - w_of
    row_w = np.bincount(r_of, weights=w_of, minlength=m).astype(np.int64)
    row_w0 = np.concatenate(([0], np.cumsum(row_w)[:-1])) if m else np.zeros(0, np.int64)
    p = s_ptr[r_of] + (wcum - row_w0[r_of])
    s_col[p] = pos_col[j_of]
    s_val[p] = A.data
    two = w_of == 2
    s_col[p[two] + 1] = pos_col[j_of[two]] + 1
    s_val[p[two] + 1] = -A.data[two]
    ri = np.nonzero(ineq)[0]
    s_col[s_ptr[ri + 1] - 1] = n_struct + ineq_idx[ri]
    s_val[s_ptr[ri + 1] - 1] = coef_row[ri]
    br = m + np.arange(n_bound)
    q = s_ptr[br]
    s_col[q], s_val[q] = pos_col[bound_j], 1.0
    split_b = ~fin[bound_j]
    s_col[q[split_b] + 1], s_val[q[split_b] + 1] = pos_col[bound_j[split_b]] + 1, -1.0
    s_col[s_ptr[br + 1] - 1] = n_struct + n_ineq + np.arange(n_bound)
    s_val[s_ptr[br + 1] - 1] = 1.0
    A_std = sp.csr_matrix((s_val, s_col.astype(np.int32), s_ptr.astype(np.int32)), shape=(m_std, n_std))

    # b_work[col_rows] -= col_vals * lo for columns j ascending (lp_core.py:281-283):
    # per row, its shifted entries in column order -- applied in rounds k = 0, 1, ...
    b_work = np.asarray(g.rhs, dtype=float).copy()
    sh = fin[j_of] & (lo[j_of] != 0.0)
    if sh.any():
        r_s, j_s, a_s = r_of[sh], j_of[sh], A.data[sh]
        rank = np.arange(r_s.size) - np.searchsorted(r_s, r_s, side="left")
        for k in range(int(rank.max()) + 1):
            sel = rank == k
            b_work[r_s[sel]] = b_work[r_s[sel]] - a_s[sel] * lo[j_s[sel]]
    b_extra = up[bound_j] - shifts[bound_j]                         # lp_core.py:336
    b_std = np.concatenate((b_work, b_extra))
    c_std = np.zeros(n_std)
    c_std[pos_col] = c
    c_std[pos_col[~fin] + 1] = -c[~fin]
    terms = c[fin & (lo != 0.0)] * lo[fin & (lo != 0.0)]            # lp_core.py:284
    obj_shift = float(np.add.accumulate(np.concatenate(([float(getattr(g, "obj_offset", 0.0))],
                                                        terms)))[-1])
    slack_of_row = np.full(m_std, -1, dtype=np.int64)
    slack_coef = np.zeros(m_std)
    slack_of_row[ri] = n_struct + ineq_idx[ri]
    slack_coef[ri] = coef_row[ri]
    slack_of_row[br] = n_struct + n_ineq + np.arange(n_bound)
    slack_coef[br] = 1.0
    bound_var = np.full(m_std, -1, dtype=np.int64)
    bound_var[br] = bound_j
    fmap = StandardFormMap(n, m, n_std, m_std, obj_shift, shifts, pos_col, neg_col,
                           slack_of_row, slack_coef, bound_var)
    return Model(A_std, b_std, c_std), fmap


# ----------------------------------------------------------------- finishing (§8(f) row 3)


def _as_float_array(v, n):
    """lp_core.py:31-35."""
    a = np.asarray(v, dtype=float).ravel()
    if a.size != n:
        raise InvalidModelError(f"expected array of length {n}, got {a.size}")
    return a


def unscale_point(row_scale, col_scale, pt: KktPoint) -> KktPoint:
    """transform.py:87-93: x = C x_s, y = R y_s, z = z_s / C."""
    return KktPoint(col_scale * pt.x, row_scale * pt.y, pt.z / col_scale)


def restrict_point(g, fmap: StandardFormMap, pt: KktPoint):
    """lp_core.py:371-385 -> (x, y, z) over the general model."""
    if pt.x.size != fmap.n_std or pt.y.size != fmap.m_std:
        raise InvalidModelError("point does not match the standard form of this map")
    x = pt.x[fmap.pos_col] + fmap.shifts
    split = fmap.neg_col >= 0
    if split.any():
        x = np.where(split, pt.x[fmap.pos_col] - pt.x[np.maximum(fmap.neg_col, 0)], x)
    y = pt.y[: fmap.m_general].copy()
    z = g.c - sp.csr_matrix(g.A, dtype=float).T @ y
    return x, y, np.asarray(z)


def lift_point(g, p, fmap: StandardFormMap, x, y) -> KktPoint:
    """lp_core.py:388-427.  The slack loop's builtin max(0.0, r/coef) and the
    bound-row min(0.0, z) are restated elementwise with their semantics
    (NaN -> 0.0, -0.0 -> 0.0)."""
    x = _as_float_array(x, fmap.n_general)
    y = _as_float_array(y, fmap.m_general)
    p = Model.wrap(p)
    x_std = np.zeros(fmap.n_std)
    shifted = x - fmap.shifts
    split = fmap.neg_col >= 0
    x_std[fmap.pos_col] = np.maximum(shifted, 0.0)
    if split.any():
        x_std[fmap.neg_col[split]] = np.maximum(-shifted[split], 0.0)
    r = p.b - p.A @ x_std
    rows = np.nonzero(fmap.slack_of_row >= 0)[0]
    v = r[rows] / fmap.slack_coef[rows]
    x_std[fmap.slack_of_row[rows]] = np.where(v > 0.0, v, 0.0)
    y_std = np.zeros(fmap.m_std)
    y_std[: fmap.m_general] = y
    brows = np.nonzero(fmap.bound_var >= 0)[0]
    if brows.size:
        z_gen = g.c - sp.csr_matrix(g.A, dtype=float).T @ y
        zb = z_gen[fmap.bound_var[brows]]
        y_std[brows] = np.where(zb < 0.0, zb, 0.0)
    z_std = np.maximum(0.0, p.c - p.at_y(y_std))
    return KktPoint(x_std, y_std, z_std)


def evaluate_general_point(g, x, y):
    """lp_core.py:488-492."""
    p, fmap = to_standard_form(g)
    pt = lift_point(g, p, fmap, x, y)
    return violation_summary(p, pt)


# ----------------------------------------------------------------- IPM hand-off (§8(f) row 4)


def mu_target(x, z, n: int, mu_min: float) -> float:
    """warmstart.py:62-68."""
    x = np.asarray(x, dtype=float)
    z = np.asarray(z, dtype=float)
    if x.size != n or z.size != n or n < 1:
        raise InvalidModelError("x and z must both have length n >= 1")
    return max(float(x @ z) / n, mu_min)


def center_toward_target(x, z, mu: float, alpha_min: float, delta_max: float):
    """warmstart.py:71-96 (same numpy ufuncs, same order)."""
    a, d = alpha_min, delta_max
    xp = np.maximum(np.asarray(x, dtype=float), a)
    zp = np.maximum(np.asarray(z, dtype=float), a)
    x_first = xp < zp
    x1 = np.clip(mu / zp, xp - d, xp + d)
    z1 = np.clip(mu / x1, zp - d, zp + d)
    z2 = np.clip(mu / xp, zp - d, zp + d)
    x2 = np.clip(mu / z2, xp - d, xp + d)
    return np.maximum(np.where(x_first, x1, x2), a), np.maximum(np.where(x_first, z1, z2), a)


def centered_start(pt: KktPoint, mu_min=1e-6, alpha_min=1e-6, delta_max=1e-4) -> KktPoint:
    """warmstart.py:99-107 (WarmStartParams defaults, warmstart.py:47-52)."""
    mu = mu_target(pt.x, pt.z, pt.x.size, mu_min)
    xn, zn = center_toward_target(pt.x, pt.z, mu, alpha_min, delta_max)
    return KktPoint(xn, pt.y.copy(), zn)
