"""numpy/scipy restatement of the reference Ruiz equilibration (TEST INFRASTRUCTURE).

Follows /root/reference/pkg/src/hybridlp/transform.py:35-77 with the same
scipy operations, so row/column scales and the scaled matrix are
bit-identical to the reference on the same scipy build.  Used to prepare
parity inputs (the reference hands run_pdhg a Ruiz-scaled model,
warmstart.py:178-197) and as the checker for the device equilibration.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .pdhg_port import Model


class ScalingError(ValueError):
    """transform.py:22-23."""


@dataclass
class ScalingInfo:
    """transform.py:26-32."""

    row_scale: np.ndarray
    col_scale: np.ndarray
    applied_iterations: int


def ruiz_equilibrate(p, max_iters: int = 20, tol: float = 1e-2):
    """transform.py:35-77. Returns (Model, ScalingInfo)."""
    A = p.A.copy().tocsr()
    m, n = A.shape
    row_nnz = np.diff(A.indptr)
    if (row_nnz == 0).any():
        i = int(np.nonzero(row_nnz == 0)[0][0])
        raise ScalingError(f"row {i} has no nonzero entries")
    col_nnz = np.diff(A.tocsc().indptr)
    if (col_nnz == 0).any():
        j = int(np.nonzero(col_nnz == 0)[0][0])
        raise ScalingError(f"column {j} has no nonzero entries")

    row_scale = np.ones(m)
    col_scale = np.ones(n)
    lo, hi = 1.0 / (1.0 + tol), 1.0 + tol
    applied = 0
    for _ in range(max_iters):
        absA = abs(A)
        row_norm = absA.max(axis=1).toarray().ravel()
        col_norm = absA.max(axis=0).toarray().ravel()
        if (
            np.all((row_norm >= lo) & (row_norm <= hi))
            and np.all((col_norm >= lo) & (col_norm <= hi))
        ):
            break
        r = 1.0 / np.sqrt(row_norm)
        c = 1.0 / np.sqrt(col_norm)
        A = sp.diags(r) @ A @ sp.diags(c)
        row_scale *= r
        col_scale *= c
        applied += 1

    scaled = Model(A.tocsr(), row_scale * np.asarray(p.b, dtype=float),
                   col_scale * np.asarray(p.c, dtype=float))
    return scaled, ScalingInfo(row_scale, col_scale, applied)
