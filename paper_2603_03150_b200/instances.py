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


# ----------------------------------------------------------------- general-form instances

EQ_S, LE_S, GE_S = "=", "<=", ">="   # hybridlp.lp_core.EQ/LE/GE (lp_core.py:22-25)


@dataclass
class GeneralInstance:
    """A general LP ``min c'x + obj_offset, A x (<=,>=,=) rhs, lower <= x <= upper``.

    Duck-types the reference ``GeneralLp`` (lp_core.py:38-103): the fields the
    standard-form builder reads, plus ``validate`` with the reference's
    checks and messages.  ``to_reference()`` builds the real GeneralLp when
    hybridlp is importable.
    """

    name: str
    c: np.ndarray
    A: sp.csr_matrix
    senses: list
    rhs: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    obj_offset: float = 0.0
    x_star: np.ndarray | None = None
    y_star: np.ndarray | None = None

    @property
    def n_vars(self) -> int:
        return self.A.shape[1]

    @property
    def n_rows(self) -> int:
        return self.A.shape[0]

    def validate(self) -> None:
        from .lp_types import resolve

        err = resolve().InvalidModelError
        if not np.all(np.isfinite(self.c)):
            raise err("objective coefficients must be finite")
        if not np.all(np.isfinite(self.rhs)):
            raise err("right-hand sides must be finite")
        if not np.all(np.isfinite(self.A.data)):
            raise err("matrix entries must be finite")
        bad = [s for s in set(self.senses) if s not in (LE_S, GE_S, EQ_S)]
        if bad:
            raise err(f"unknown row sense {bad[0]!r}")
        crossed = np.nonzero(self.lower > self.upper)[0]
        if crossed.size:
            j = int(crossed[0])
            raise err(f"variable {j} has lower bound {self.lower[j]} above upper bound {self.upper[j]}")

    def to_reference(self):
        from hybridlp import GeneralLp  # type: ignore

        return GeneralLp(c=self.c, A=self.A, senses=list(self.senses), rhs=self.rhs,
                         lower=self.lower, upper=self.upper, obj_offset=self.obj_offset)


def config1_general(scale: float = 1.0, seed: int = 1, mean_len: float = 10.0) -> GeneralInstance:
    """BASELINE config 1: bounded-variable LP, general form.

    m=50k EQ rows x n=100k columns; row lengths lognormal (arithmetic mean
    ``mean_len``, log-sigma 1) clipped to [1, 2000]; columns uniform, values
    N(0,1), >= 1 entry per row and column.  Bounds l=0, u~U(1,10); 10% of
    the columns are free.  Planted optimum: x* interior on 40% of the
    columns (all free columns plus a third of the bounded ones), at l or u
    (half each) on the rest; y*~N(0,1); z* >= 0 at l, <= 0 at u, 0 where
    interior; c = A'y* + z*, b = A x*.  ``mean_len`` = 10 as the config
    states (~0.5M nnz at full size; the config's "~1M" needs 20).
    """
    rng = np.random.default_rng(seed)
    m = max(int(50_000 * scale), 4)
    n = 2 * m
    sigma = 1.0
    mu = np.log(mean_len) - 0.5 * sigma * sigma
    lens = np.clip(np.rint(rng.lognormal(mu, sigma, m)), 1, 2000).astype(np.int64)
    lens = np.minimum(lens, n)
    nnz = int(lens.sum())
    rows = np.repeat(np.arange(m, dtype=np.int64), lens)
    cols = rng.integers(0, n, nnz, dtype=np.int64)
    vals = rng.standard_normal(nnz)
    rows, cols, vals = _cover_empty(rows, cols, vals, m, n, rng)
    A = _csr_from_rows(rows, cols, vals, m, n)
    free = rng.random(n) < 0.1
    upper = np.where(free, np.inf, rng.uniform(1.0, 10.0, n))
    lower = np.where(free, -np.inf, 0.0)
    u = rng.random(n)
    interior = free | (u < 1.0 / 3.0)
    at_upper = ~interior & (u >= 2.0 / 3.0)
    at_lower = ~interior & ~at_upper
    x_star = np.zeros(n)
    xi = rng.random(n)
    x_star[interior & ~free] = (0.05 + 0.9 * xi[interior & ~free]) * upper[interior & ~free]
    x_star[free] = rng.standard_normal(int(free.sum()))
    x_star[at_upper] = upper[at_upper]
    y_star = rng.standard_normal(m)
    zmag = rng.uniform(0.0, 1.0, n)
    z_star = np.where(at_lower, zmag, np.where(at_upper, -zmag, 0.0))
    rhs = A @ x_star
    c = A.T @ y_star + z_star
    return GeneralInstance(f"config1_s{scale:g}", c, A, [EQ_S] * m, rhs, lower, upper,
                           x_star=x_star, y_star=y_star)


def grid_arcs(R: int):
    """Directed 4-neighbour grid of R x R nodes, arcs both ways: (tail, head)."""
    idx = np.arange(R * R, dtype=np.int64).reshape(R, R)
    h0, h1 = idx[:, :-1].ravel(), idx[:, 1:].ravel()
    v0, v1 = idx[:-1, :].ravel(), idx[1:, :].ravel()
    tail = np.concatenate([h0, h1, v0, v1])
    head = np.concatenate([h1, h0, v1, v0])
    return tail, head


def config3_general(scale: float = 1.0, seed: int = 3, K: int = 8) -> GeneralInstance:
    """BASELINE config 3: multicommodity flow on a directed R x R grid, general form.

    R = 300*sqrt(scale) (358,800 arcs at full size), K commodities.  Columns
    f[k, a] >= 0 (commodity-major); rows: flow conservation per (commodity,
    node), ``out - in = supply`` (EQ, entries +-1), then one capacity row per
    arc ``sum_k f[k, a] <= cap_a`` (LE, gets a slack column).  cap ~ U{1..100},
    arc cost ~ U{1..10} shared by the commodities; A's values are integers
    stored as fp64.  Supplies are integer and balanced per commodity; drawn
    i.i.d. U(-50, 50) per node they make the LP infeasible (HiGHS, R = 30 and
    60), so they are the node divergences of a random integer
    flow f0[k, a] ~ U{0..floor(cap_a/K)} -- feasible by construction, range
    about +-40.
    """
    rng = np.random.default_rng(seed)
    R = max(int(round(300 * np.sqrt(scale))), 3)
    V = R * R
    tail, head = grid_arcs(R)
    E = tail.size
    cap = rng.integers(1, 101, E).astype(np.float64)
    cost = rng.integers(1, 11, E).astype(np.float64)
    f0 = np.floor(rng.random((K, E)) * (np.floor(cap / K) + 1.0))
    supply = np.zeros((K, V))
    for k in range(K):
        supply[k] = (np.bincount(tail, weights=f0[k], minlength=V)
                     - np.bincount(head, weights=f0[k], minlength=V))
    # conservation rows: row k*V + v; column k*E + a has +1 at tail, -1 at head
    kk = np.repeat(np.arange(K, dtype=np.int64), E)
    aa = np.tile(np.arange(E, dtype=np.int64), K)
    colid = kk * E + aa
    r_out = kk * V + tail[aa]
    r_in = kk * V + head[aa]
    r_cap = K * V + aa
    rows = np.concatenate([r_out, r_in, r_cap])
    cols = np.concatenate([colid, colid, colid])
    vals = np.concatenate([np.ones(colid.size), -np.ones(colid.size), np.ones(colid.size)])
    m, n = K * V + E, K * E
    A = _csr_from_rows(rows, cols, vals, m, n)
    senses = [EQ_S] * (K * V) + [LE_S] * E
    rhs = np.concatenate([supply.ravel(), cap])
    c = np.tile(cost, K)
    return GeneralInstance(f"config3_s{scale:g}", c, A, senses, rhs, np.zeros(n), np.full(n, np.inf),
                           x_star=f0.ravel())
