"""Pin the CPU oracle (oracle/pdhg_port.py) against the reference's own outputs.

The golden files were produced by running the real reference
(/root/reference/pkg/src/hybridlp) -- see oracle/make_golden.py.  With the
same numpy/scipy build the restatement must be bit-identical; otherwise
agreement to rounding is required.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle.pdhg_port import Model


def _model(gm):
    return Model(gm.A, gm.b, gm.c)


def _eq(a, b, gm, rtol=1e-12):
    if gm.same_numerics:
        np.testing.assert_array_equal(a, b)
    else:
        np.testing.assert_allclose(a, b, rtol=rtol, atol=1e-14)


def test_opnorm_matches_reference(golden):
    lam = oracle.estimate_opnorm(golden.A, seed=0)
    _eq(np.array(lam), golden.g["opnorm_seed0"], golden)


def test_spmv_matches_reference(golden):
    p = _model(golden)
    _eq(p.A @ golden.g["spmv_v"], golden.g["spmv_Av"], golden)
    _eq(p.at_y(golden.g["spmv_w"]), golden.g["spmv_Atw"], golden)


def test_first_iterates_match_reference(golden):
    p = _model(golden)
    ks = set(int(k) for k in golden.g["it_k"])
    rec = {}

    def on_step(st):
        if st.iterations in ks:
            rec[st.iterations] = (st.x.copy(), st.y.copy(), st.avg_x.copy(), st.avg_y.copy(),
                                  st.omega, st.restarts)

    oracle.run_pdhg(p, oracle.PdhgParams(eps_rel=1e-12, max_kkt_passes=100), on_step=on_step)
    g = golden.g
    for j, k in enumerate(g["it_k"]):
        x, y, ax, ay, om, rs = rec[int(k)]
        _eq(x, g["it_x"][j], golden)
        _eq(y, g["it_y"][j], golden)
        _eq(ax, g["it_avgx"][j], golden)
        _eq(ay, g["it_avgy"][j], golden)
        assert om == pytest.approx(float(g["it_omega"][j]), rel=1e-12)
        assert rs == int(g["it_restarts"][j])


@pytest.mark.parametrize("tag,eps,limit", [("e4", 1e-4, 200_000), ("e6", 1e-6, 200_000),
                                           ("lim128", 1e-12, 128), ("lim200", 1e-12, 200)])
def test_full_run_matches_reference(golden, tag, eps, limit):
    r = golden.run(tag)
    pt, st = oracle.run_pdhg(_model(golden), oracle.PdhgParams(eps_rel=eps, max_kkt_passes=limit))
    assert st.status.value == str(r["status"])
    assert st.iterations == int(r["iterations"])
    assert st.restarts == int(r["restarts"])
    t = st.termination
    _eq(np.array([t.primal_lhs, t.primal_rhs, t.dual_lhs, t.dual_rhs, t.gap_lhs, t.gap_rhs]),
        r["term"], golden, rtol=1e-9)
    _eq(pt.x, r["x"], golden, rtol=1e-9)
    _eq(pt.y, r["y"], golden, rtol=1e-9)
    _eq(pt.z, r["z"], golden, rtol=1e-9)


def test_e8_runs_where_recorded(golden):
    r = golden.run("e8")
    if not r:
        pytest.skip("no 1e-8 run recorded for this size")
    pt, st = oracle.run_pdhg(_model(golden), oracle.PdhgParams(eps_rel=1e-8))
    assert st.iterations == int(r["iterations"])
    assert st.status.value == str(r["status"])
