"""Instance I/O for the path's inputs: a .npz CSR format.

The reference reads models through its MPS parser (out of scope) and builds
them in memory; at config 4's 200M entries neither MPS text nor a Python
builder is practical.  This format stores the arrays the path consumes:

* standard form (``StandardLp``, lp_core.py:106-142): the CSR arrays of A
  (indptr, indices, data), b, c;
* general form (``GeneralLp``, lp_core.py:38-103): the CSR arrays of A, row
  senses as one code per row ("=", "<=", ">=", the reference's
  lp_core.py:22-25 constants), rhs, lower, upper, c, obj_offset, and
  optional row / column names.

Files are written uncompressed (``np.savez``: each array is one sequential
read on load).  The loaded model is the reference's own class when hybridlp
is importable, else this package's mirror.  A round trip is bit-exact
(tests/test_lpio.py).
"""

from __future__ import annotations

import json

import numpy as np
import scipy.sparse as sp

FORMAT = "pdhg-b200-lp/1"
_SENSES = ("=", "<=", ">=")   # code 0, 1, 2


def _csr_arrays(A):
    A = sp.csr_matrix(A)
    return {"A_indptr": np.asarray(A.indptr), "A_indices": np.asarray(A.indices),
            "A_data": np.asarray(A.data, dtype=np.float64),
            "A_shape": np.asarray(A.shape, dtype=np.int64)}


def _csr_from(z) -> sp.csr_matrix:
    m, n = (int(v) for v in z["A_shape"])
    return sp.csr_matrix((z["A_data"], z["A_indices"], z["A_indptr"]), shape=(m, n))


def _header(kind: str, **extra) -> np.ndarray:
    return np.frombuffer(json.dumps({"format": FORMAT, "kind": kind, **extra}).encode(), dtype=np.uint8)


def _check(z, kind: str) -> dict:
    if "header" not in z.files:
        raise ValueError("not a pdhg-b200 LP file (no header)")
    h = json.loads(bytes(np.asarray(z["header"])).decode())
    if h.get("format") != FORMAT:
        raise ValueError(f"unsupported LP file format {h.get('format')!r}")
    if h.get("kind") != kind:
        raise ValueError(f"file holds a {h.get('kind')} LP, not a {kind} one")
    return h


def save_standard(path, p) -> None:
    """Write StandardLp-like ``p`` (A, b, c) to ``path`` (.npz)."""
    np.savez(path, header=_header("standard"), b=np.asarray(p.b, dtype=np.float64),
             c=np.asarray(p.c, dtype=np.float64), **_csr_arrays(p.A))


def load_standard(path):
    """Read a standard-form LP written by save_standard."""
    from .lp_types import resolve

    with np.load(path, allow_pickle=False) as z:
        _check(z, "standard")
        A = _csr_from(z)
        b, c = np.array(z["b"]), np.array(z["c"])
    return resolve().StandardLp(A, b, c)


def save_general(path, g) -> None:
    """Write GeneralLp-like ``g`` to ``path`` (.npz)."""
    codes = np.fromiter((_SENSES.index(s) for s in g.senses), dtype=np.uint8, count=len(g.senses))
    names = {}
    for key in ("row_names", "col_names"):
        v = getattr(g, key, None)
        if v is not None:
            names[key] = np.asarray(list(v), dtype=str)
    np.savez(path, header=_header("general", obj_offset=float(getattr(g, "obj_offset", 0.0))),
             senses=codes, rhs=np.asarray(g.rhs, dtype=np.float64), lower=np.asarray(g.lower, dtype=np.float64),
             upper=np.asarray(g.upper, dtype=np.float64), c=np.asarray(g.c, dtype=np.float64),
             **names, **_csr_arrays(g.A))


def load_general(path):
    """Read a general-form LP written by save_general: the reference's
    GeneralLp when hybridlp is importable, else instances.GeneralInstance."""
    with np.load(path, allow_pickle=False) as z:
        h = _check(z, "general")
        A = _csr_from(z)
        arrays = {k: np.array(z[k]) for k in ("rhs", "lower", "upper", "c")}
        senses = [_SENSES[int(k)] for k in np.asarray(z["senses"])]
        names = {k: [str(s) for s in z[k]] for k in ("row_names", "col_names") if k in z.files}
    try:
        from hybridlp import GeneralLp  # type: ignore
    except ImportError:
        from .instances import GeneralInstance

        return GeneralInstance(name=str(path), c=arrays["c"], A=A, senses=senses, rhs=arrays["rhs"],
                               lower=arrays["lower"], upper=arrays["upper"], obj_offset=h["obj_offset"])
    return GeneralLp(c=arrays["c"], A=A, senses=senses, rhs=arrays["rhs"], lower=arrays["lower"],
                     upper=arrays["upper"], obj_offset=h["obj_offset"], **names)
