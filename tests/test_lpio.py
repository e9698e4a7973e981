"""The .npz instance format (paper_2603_03150_b200/lpio.py): bit-exact round
trips of standard- and general-form models, and the format checks."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden


def _same_csr(A, B):
    A, B = A.tocsr(), B.tocsr()
    assert A.shape == B.shape
    for k in ("indptr", "indices", "data"):
        assert getattr(A, k).tobytes() == getattr(B, k).tobytes()


def test_standard_round_trip(tmp_path):
    from paper_2603_03150_b200 import lpio

    gm = load_golden("config0_s0")
    f = tmp_path / "m.npz"
    lpio.save_standard(f, gm)
    p = lpio.load_standard(f)
    _same_csr(p.A, gm.A)
    assert np.asarray(p.b).tobytes() == np.asarray(gm.b, dtype=float).tobytes()
    assert np.asarray(p.c).tobytes() == np.asarray(gm.c, dtype=float).tobytes()


def test_general_round_trip_and_standard_form(tmp_path):
    from oracle.stdform_port import to_standard_form
    from paper_2603_03150_b200 import lpio
    from paper_2603_03150_b200.instances import config1_general

    g = config1_general(0.02, seed=3)
    g.obj_offset = 1.25
    f = tmp_path / "g.npz"
    lpio.save_general(f, g)
    h = lpio.load_general(f)
    _same_csr(h.A, g.A)
    assert list(h.senses) == list(g.senses) and float(h.obj_offset) == 1.25
    for k in ("rhs", "lower", "upper", "c"):
        assert np.asarray(getattr(h, k)).tobytes() == np.asarray(getattr(g, k), dtype=float).tobytes()
    (p1, m1), (p2, m2) = to_standard_form(g), to_standard_form(h)
    _same_csr(p1.A, p2.A)
    assert p1.b.tobytes() == p2.b.tobytes() and p1.c.tobytes() == p2.c.tobytes()


def test_format_checks(tmp_path):
    from paper_2603_03150_b200 import lpio

    gm = load_golden("config0_s0")
    f = tmp_path / "m.npz"
    lpio.save_standard(f, gm)
    with pytest.raises(ValueError, match="not a general one"):
        lpio.load_general(f)
    np.savez(tmp_path / "x.npz", a=np.zeros(3))
    with pytest.raises(ValueError, match="no header"):
        lpio.load_standard(tmp_path / "x.npz")
