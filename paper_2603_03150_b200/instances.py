"""Seeded synthetic LP instances for the five BASELINE.json configurations.

These are the inputs the parity tests and bench.py feed to BOTH the device
engine and the CPU oracle, so both sides read bit-identical arrays.  The
paper's own benchmark sets (Mittelmann LP set, the 2,298-model set) are not
available here; these seeded instances stand in for them, with the shapes,
sizes and value distributions BASELINE.json states.

All generators use numpy's PCG64 ``default_rng(seed)`` and return CSR
matrices with sorted, duplicate-free column indices and at least one stored
entry in every row and column (Ruiz equilibration, transform.py:47-54,
rejects empty rows and columns).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass
class Instance:
    """A standard-form LP ``min c'x, Ax=b, x>=0`` plus its planted optimum.

    Duck-types the reference ``StandardLp`` (lp_core.py:106-142): ``A`` is a
    float64 CSR matrix, ``b`` and ``c`` are float64 vectors.
    """

    name: str
    A: sp.csr_matrix
    b: np.ndarray
    c: np.ndarray
    x_star: np.ndarray | None = None
    y_star: np.ndarray | None = None

    @property
    def m(self) -> int:
        return self.A.shape[0]

    @property
    def n(self) -> int:
        return self.A.shape[1]

    @property
    def nnz(self) -> int:
        return int(self.A.nnz)


def _csr_from_rows(rows: np.ndarray, cols: np.ndarray, vals: np.ndarray, m: int, n: int):
    """CSR from row-grouped triplets; sorts columns within rows, drops duplicates."""
    key = rows.astype(np.int64) * n + cols.astype(np.int64)
    order = np.argsort(key, kind="stable")
    key = key[order]
    keep = np.ones(key.size, dtype=bool)
    keep[1:] = key[1:] != key[:-1]
    key = key[keep]
    vals = vals[order][keep]
    r = key // n
    cidx = (key - r * n).astype(np.int32)
    indptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=m), out=indptr[1:])
    if indptr[-1] < 2**31:
        indptr = indptr.astype(np.int32)
    A = sp.csr_matrix((vals, cidx, indptr), shape=(m, n))
    A.has_sorted_indices = True
    return A


def _cover_empty(rows, cols, vals, m, n, rng):
    """Give every empty row and column one N(0,1) entry at a random position."""
    row_cnt = np.bincount(rows, minlength=m)
    col_cnt = np.bincount(cols, minlength=n)
    er = np.nonzero(row_cnt == 0)[0]
    ec = np.nonzero(col_cnt == 0)[0]
    add_r = [er, rng.integers(0, m, ec.size)]
    add_c = [rng.integers(0, n, er.size), ec]
    add_v = rng.standard_normal(er.size + ec.size)
    if er.size + ec.size == 0:
        return rows, cols, vals
    rows = np.concatenate([rows, add_r[0], add_r[1]])
    cols = np.concatenate([cols, add_c[0], add_c[1]])
    vals = np.concatenate([vals, add_v])
    return rows, cols, vals


def _plant(A: sp.csr_matrix, rng, frac_support: float = 0.5):
    """Planted KKT triple as in BASELINE config 0: x* U(0,1) on a random half
    of the columns, y* ~ N(0,1), z* U(0,1) exactly where x* = 0;
    b = A x*, c = A'y* + z*."""
    m, n = A.shape
    support = rng.random(n) < frac_support
    x_star = np.where(support, rng.random(n), 0.0)
    y_star = rng.standard_normal(m)
    z_star = np.where(support, 0.0, rng.random(n))
    b = A @ x_star
    c = A.T @ y_star + z_star
    return b, c, x_star, y_star


def config0_general(seed: int = 0):
    """BASELINE config 0 as a general LP (EQ rows, 0 <= x < inf), the form the
    reference's ``hybrid_solve`` pipeline starts from.

    Returns (A csr, b, c, x_star, y_star); m=500, n=1000, 1% density.
    """
    rng = np.random.default_rng(seed)
    m, n = 500, 1000
    pos = rng.choice(m * n, size=m * n // 100, replace=False)
    rows, cols = pos // n, pos % n
    vals = rng.standard_normal(pos.size)
    rows, cols, vals = _cover_empty(rows, cols, vals, m, n, rng)
    A = _csr_from_rows(rows, cols, vals, m, n)
    b, c, xs, ys = _plant(A, rng)
    return A, b, c, xs, ys


def lognormal_rows(m: int, n: int, mean_len: float, sigma: float, max_len: int,
                   seed: int, band_frac: float = 0.0, band_half: int = 0,
                   name: str = "lognormal") -> Instance:
    """Planted standard-form LP with lognormal row lengths.

    Row lengths: lognormal with arithmetic mean ``mean_len`` and log-sigma
    ``sigma``, rounded, clipped to [1, max_len].  Column of each entry:
    with probability ``band_frac`` uniform within +-band_half of the row's
    diagonal i*n/m (wrapped modulo n -- clamping would pile entries onto
    column 0), otherwise uniform.  Values N(0,1).
    """
    rng = np.random.default_rng(seed)
    mu = np.log(mean_len) - 0.5 * sigma * sigma
    lens = np.clip(np.rint(rng.lognormal(mu, sigma, m)), 1, max_len).astype(np.int64)
    nnz = int(lens.sum())
    rows = np.repeat(np.arange(m, dtype=np.int64), lens)
    cols = rng.integers(0, n, nnz, dtype=np.int64)
    if band_frac > 0.0:
        band = rng.random(nnz) < band_frac
        nb = int(band.sum())
        centre = (rows[band] * n) // m
        off = rng.integers(-band_half, band_half + 1, nb, dtype=np.int64)
        cols[band] = (centre + off) % n
    vals = rng.standard_normal(nnz)
    rows, cols, vals = _cover_empty(rows, cols, vals, m, n, rng)
    A = _csr_from_rows(rows, cols, vals, m, n)
    b, c, xs, ys = _plant(A, rng)
    return Instance(name, A, b, c, xs, ys)


def config4(scale: float = 1.0, seed: int = 4) -> Instance:
    """BASELINE config 4: 5M x 10M, lognormal rows (mean 40, sigma 0.8),
    70% of columns within +-50k of the diagonal (wrapped), 30% uniform,
    N(0,1) values, planted optimum.  ``scale`` shrinks m, n and the band
    proportionally (1.0 = the full 200M-nnz instance)."""
    m = max(int(5_000_000 * scale), 2)
    n = 2 * m
    half = max(int(50_000 * scale), 1)
    return lognormal_rows(m, n, 40.0, 0.8, 2000, seed, band_frac=0.7, band_half=half,
                          name=f"config4_s{scale:g}")


def config2(scale: float = 1.0, seed: int = 2, k_min: int = 6) -> Instance:
    """BASELINE config 2 (heavy-tailed rows), built directly in standard form.

    500k x 1M structural columns; 70% EQ rows, 30% <= rows that get a slack
    column each (so n_std = n + 0.3 m).  Row nnz follow a discrete power law
    p(k) ~ k^-2.1 on [k_min, 50k] (k_min=6 gives ~20M nnz).
    Values N(0,1) times a per-row U(0.1, 10).  The optimum is planted in the
    standard form including the slack columns.
    """
    rng = np.random.default_rng(seed)
    m = max(int(500_000 * scale), 4)
    n = 2 * m
    kmax = max(min(50_000, int(50_000 * scale)), k_min + 1)
    ks = np.arange(k_min, kmax + 1, dtype=np.float64)
    p = ks ** -2.1
    p /= p.sum()
    lens = rng.choice(ks.astype(np.int64), size=m, p=p)
    lens = np.minimum(lens, n)
    nnz = int(lens.sum())
    rows = np.repeat(np.arange(m, dtype=np.int64), lens)
    cols = rng.integers(0, n, nnz, dtype=np.int64)
    vals = rng.standard_normal(nnz) * np.repeat(rng.uniform(0.1, 10.0, m), lens)
    ineq = np.nonzero(rng.random(m) < 0.3)[0]
    slack_cols = n + np.arange(ineq.size, dtype=np.int64)
    rows = np.concatenate([rows, ineq])
    cols = np.concatenate([cols, slack_cols])
    vals = np.concatenate([vals, np.ones(ineq.size)])
    n_std = n + ineq.size
    rows, cols, vals = _cover_empty(rows, cols, vals, m, n_std, rng)
    A = _csr_from_rows(rows, cols, vals, m, n_std)
    b, c, xs, ys = _plant(A, rng)
    return Instance(f"config2_s{scale:g}", A, b, c, xs, ys)
