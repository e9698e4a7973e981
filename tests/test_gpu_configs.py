"""BASELINE configs 1 and 3 through the device pipeline (GPU).

general LP -> device standard form (csrc/stdform.cu) -> device Ruiz
(csrc/ruiz.cu) -> run_pdhg (sm_100a step kernels) -> device finishing
(csrc/finish.cu), against
  * the oracle pipeline iterate by iterate at reduced size (1e-9 relative,
    first 100 iterates including the iteration-64 check), and
  * the REAL reference's full-size runs (tests/golden/run_*.json, written by
    oracle/make_golden_runs.py in the build container): status, iteration
    count, restarts and objective; the returned point re-checked by the
    oracle's termination test at full size.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from oracle import stdform_port as SF
from oracle.pdhg_port import KktPoint, Model
from oracle.ruiz_port import ruiz_equilibrate as ruiz_port

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


@pytest.fixture(scope="module")
def eng():
    import paper_2603_03150_b200 as e

    return e


def _rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(1.0, float(np.max(np.abs(b)))))


def _standard(which, scale):
    from paper_2603_03150_b200.instances import config2

    return config2(scale)


def _general(which, scale, seed=None):
    from paper_2603_03150_b200.instances import config1_general, config3_general

    f = config1_general if which == "config1" else config3_general
    return f(scale) if seed is None else f(scale, seed=seed)


def _device_pipeline(eng, g):
    p, fmap = eng.to_standard_form(g)
    scaled, info = eng.ruiz_equilibrate(p)
    return p, fmap, scaled, info


@pytest.mark.parametrize("which,scale", [("config1", 0.02), ("config3", 0.01)])
def test_first_iterates_match_oracle(eng, which, scale):
    from paper_2603_03150_b200 import _native as N

    T = eng.types()
    g = _general(which, scale)
    p, fmap, scaled, info = _device_pipeline(eng, g)
    q, _ = SF.to_standard_form(g)
    qs, _ = ruiz_port(q)
    assert sp.csr_matrix(scaled.A).data.tobytes() == qs.A.data.tobytes()
    keep = {1, 2, 63, 64, 65, 100}
    rec = {}
    oracle.run_pdhg(Model(qs.A, qs.b, qs.c), oracle.PdhgParams(eps_rel=1e-12, max_kkt_passes=100),
                    on_step=lambda st: rec.__setitem__(st.iterations, (st.x.copy(), st.y.copy(),
                                                                        st.avg_x.copy(), st.avg_y.copy()))
                    if st.iterations in keep else None)
    opts = eng.GpuOptions()
    for k in sorted(keep):
        ce = 10**6 if k % 64 == 0 else 64
        eng.run_pdhg(scaled, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=k, check_every=ce), gpu=opts)
        dev = eng.device_lp(scaled, opts)
        x, y, _ = dev.fetch(N.PT_CUR, want_z=False)
        ax, ay, _ = dev.fetch(N.PT_AVG, want_z=False)
        ox, oy, oax, oay = rec[k]
        assert _rel(x, ox) <= 1e-9 and _rel(y, oy) <= 1e-9, k
        assert _rel(ax, oax) <= 1e-9 and _rel(ay, oay) <= 1e-9, k


@pytest.mark.parametrize("which,scale", [("config1", 1.0), ("config3", 0.1), ("config3", 1.0),
                                         ("config2", 0.1)])
def test_full_run_matches_reference(eng, which, scale):
    """Full-size run to eps_rel=1e-4 against the reference's own run."""
    path = GOLD / f"run_{which}_s{scale:g}.json"
    if not path.exists():
        pytest.skip(f"no reference run recorded for {which} scale {scale}")
    ref = json.loads(path.read_text())
    T = eng.types()
    if which == "config2":   # standard form already: device Ruiz -> PDHG
        scaled, info = eng.ruiz_equilibrate(_standard(which, scale))
    else:
        g = _general(which, scale)
        p, fmap, scaled, info = _device_pipeline(eng, g)
    assert (scaled.A.shape[0], scaled.A.shape[1], int(scaled.A.nnz)) == (ref["m_std"], ref["n_std"], ref["nnz_std"])
    pt, st = eng.run_pdhg(scaled, T.PdhgParams(eps_rel=1e-4))
    assert st.status.value == ref["status"] == "Optimal"
    it, rit = st.iterations, ref["iterations"]
    assert (it == rit) if rit < 1280 else abs(it - rit) <= 0.05 * rit, (it, rit)
    assert st.restarts == ref["restarts"], (st.restarts, ref["restarts"])
    obj = float(scaled.c @ pt.x)
    assert abs(obj - ref["objective_scaled"]) <= 1e-6 * max(1.0, abs(ref["objective_scaled"]))
    # size-independent: the returned point passes the oracle's termination test
    t = oracle.check_relative_termination(Model(scaled.A, scaled.b, scaled.c),
                                          KktPoint(pt.x, pt.y, pt.z), 1e-4)
    assert t.ok
    print(f"{which} s{scale:g}: {it} iterations ({rit} reference), {st.restarts} restarts, "
          f"{st.wall_seconds:.2f}s GPU vs {ref['seconds']['run_pdhg']:.0f}s reference run_pdhg")


def test_config1_finishing_on_general_model(eng):
    """Device unscale + restrict + evaluate_general_point equal the oracle's
    on the GPU's own PDHG point (config 1, full size)."""
    from paper_2603_03150_b200 import finish

    T = eng.types()
    g = _general("config1", 1.0)
    p, fmap, scaled, info = _device_pipeline(eng, g)
    pt, st = eng.run_pdhg(scaled, T.PdhgParams(eps_rel=1e-4))
    un = finish.unscale_point(info, pt)
    oun = SF.unscale_point(info.row_scale, info.col_scale, KktPoint(pt.x, pt.y, pt.z))
    assert un.x.tobytes() == oun.x.tobytes() and un.z.tobytes() == oun.z.tobytes()
    x, y, z = finish.restrict_point(g, fmap, un)
    ox, oy, oz = SF.restrict_point(g, fmap, oun)
    assert x.tobytes() == ox.tobytes() and z.tobytes() == oz.tobytes()
    v = finish.evaluate_general_point(g, x, y)
    ov = SF.evaluate_general_point(g, ox, oy)
    assert v.primal_inf == ov.primal_inf and v.dual_inf == ov.dual_inf
    assert abs(v.rel_gap - ov.rel_gap) <= 1e-12 * max(1.0, abs(ov.rel_gap))
