"""IPM hand-off: centered_start / center_toward_target /
mu_target (warmstart.py:62-107) against the real reference's outputs
(tests/golden/center.npz, oracle/make_golden_center.py).  CPU: the oracle
restatement bit for bit; GPU: the device kernel bit for bit for a given mu,
and centered_start to rounding (x'z is a fixed-order device dot)."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import stdform_port as SF
from oracle.pdhg_port import KktPoint

Z = np.load(Path(__file__).parent / "golden" / "center.npz")


def same(a, b):
    return np.asarray(a).tobytes() == np.asarray(b).tobytes()


@pytest.mark.parametrize("k", [0, 1, 2])
def test_oracle_center_matches_reference(k):
    mu, a, d = Z[f"ct{k}_params"]
    xn, zn = SF.center_toward_target(Z["x"], Z["z"], mu, a, d)
    assert same(xn, Z[f"ct{k}_x"]) and same(zn, Z[f"ct{k}_z"])


def test_oracle_centered_start_matches_reference():
    x, z = np.nan_to_num(Z["x"], nan=1.0), np.nan_to_num(Z["z"], nan=1.0)
    cs = SF.centered_start(KktPoint(x, Z["y"], z))
    assert same(cs.x, Z["cs_x"]) and same(cs.z, Z["cs_z"]) and same(cs.y, Z["cs_y"])


@pytest.mark.gpu
@pytest.mark.parametrize("k", [0, 1, 2])
def test_device_center_is_bitwise_reference(k):
    from paper_2603_03150_b200 import finish

    mu, a, d = Z[f"ct{k}_params"]
    xn, zn = finish.center_toward_target(Z["x"], Z["z"], mu, a, d)
    assert same(xn, Z[f"ct{k}_x"]) and same(zn, Z[f"ct{k}_z"])


@pytest.mark.gpu
def test_device_centered_start_matches_reference():
    from paper_2603_03150_b200 import finish

    x, z = np.nan_to_num(Z["x"], nan=1.0), np.nan_to_num(Z["z"], nan=1.0)
    mu = finish.mu_target(x, z, x.size, 1e-6)
    assert abs(mu - float(Z["cs_mu"][0])) <= 1e-14 * abs(float(Z["cs_mu"][0]))
    cs = finish.centered_start(KktPoint(x, Z["y"], z))
    np.testing.assert_allclose(cs.x, Z["cs_x"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(cs.z, Z["cs_z"], rtol=1e-13, atol=0)
    assert same(cs.y, Z["cs_y"])
