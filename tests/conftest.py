"""Shared fixtures: golden models from tests/golden (made by oracle/make_golden.py)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpdhg_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


GOLDEN_NAMES = sorted(p.stem for p in GOLDEN.glob("*.npz")
                      if not p.stem.startswith(("ruiz_", "stdform_", "center", "full_")))
RUIZ_NAMES = sorted(p.stem for p in GOLDEN.glob("ruiz_*.npz"))


class GoldenModel:
    """A StandardLp-like model (A CSR float64, b, c) loaded from a golden file."""

    def __init__(self, name: str):
        self.name = name
        self.g = np.load(GOLDEN / f"{name}.npz")
        g = self.g
        self.A = sp.csr_matrix((g["A_data"], g["A_indices"], g["A_indptr"]),
                               shape=tuple(g["A_shape"]))
        self.b = g["b"].copy()
        self.c = g["c"].copy()

    @property
    def m(self):
        return self.A.shape[0]

    @property
    def n(self):
        return self.A.shape[1]

    def run(self, tag):
        g = self.g
        return {k[len(f"run_{tag}_"):]: g[k] for k in g.files if k.startswith(f"run_{tag}_")}

    @property
    def same_numerics(self) -> bool:
        import scipy

        return (str(self.g["numpy_version"]) == np.__version__
                and str(self.g["scipy_version"]) == scipy.__version__)


@pytest.fixture(scope="session", params=GOLDEN_NAMES)
def golden(request):
    return GoldenModel(request.param)


def load_golden(name: str) -> GoldenModel:
    return GoldenModel(name)


def experimental_build() -> bool:
    """Is the loaded library the experiment build?  (Collection-time: the
    experiment-only parametrizations are left out of the product build's run.)"""
    try:
        from paper_2603_03150_b200 import _native

        return _native.experimental()
    except Exception:
        return False


EXPERIMENTAL_BUILD = experimental_build()


def skip_unless_experimental(what: str = "layout") -> None:
    """PSR layouts, persistent periods and L2 windows exist only in the
    experiment build of the library (measured slower)."""
    from paper_2603_03150_b200 import _native

    if not _native.experimental():
        pytest.skip(f"{what}: experiment build only (PDHG_B200_LIB=tools/_libs/libpdhg_b200_exp.so)")
