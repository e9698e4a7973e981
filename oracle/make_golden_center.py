"""Golden vectors for the IPM hand-off (TEST INFRASTRUCTURE): the REAL reference's
mu_target / center_toward_target / centered_start (warmstart.py:62-107) on
seeded points including the edge values the functions branch on (zeros,
negatives, ties, values below alpha_min, moves larger than delta_max, NaN),
written to tests/golden/center.npz.  Runs only where /root/reference exists.

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_center.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[1]

import hybridlp  # noqa: E402
from hybridlp import warmstart as W  # noqa: E402


def main():
    rng = np.random.default_rng(11)
    n = 5000
    x = np.abs(rng.standard_normal(n)) * 10.0 ** rng.uniform(-9, 2, n)
    z = np.abs(rng.standard_normal(n)) * 10.0 ** rng.uniform(-9, 2, n)
    x[:50] = 0.0
    z[50:100] = 0.0
    x[100:150] = -rng.random(50)
    z[150:200] = z[200:250] = x[150:200]        # ties
    x[250:260] = 1e-7                            # below alpha_min
    x[260] = np.nan
    z[261] = np.nan
    y = rng.standard_normal(300)
    out = {"x": x, "z": z, "y": y}
    for k, (mu, a, d) in enumerate(((0.37, 1e-6, 1e-4), (1e-3, 1e-6, 1e-2), (5.0, 1e-3, 1.0))):
        xn, zn = W.center_toward_target(x, z, mu, a, d)
        out[f"ct{k}_params"] = np.array([mu, a, d])
        out[f"ct{k}_x"], out[f"ct{k}_z"] = xn, zn
    xf, zf = np.nan_to_num(x, nan=1.0), np.nan_to_num(z, nan=1.0)
    pt = hybridlp.KktPoint(xf, y, zf)
    cs = W.centered_start(pt)
    out["cs_x"], out["cs_y"], out["cs_z"] = cs.x, cs.y, cs.z
    out["cs_mu"] = np.array([W.mu_target(xf, zf, n, W.WarmStartParams().mu_min)])
    np.savez_compressed(ROOT / "tests" / "golden" / "center.npz", numpy_version=np.__version__, **out)
    print("wrote tests/golden/center.npz")


if __name__ == "__main__":
    main()
