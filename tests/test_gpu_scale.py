"""GPU parity at larger sizes (scaled BASELINE configs) against the CPU oracle,
plus size-independent properties at the full config-4 size."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import EXPERIMENTAL_BUILD, skip_unless_experimental
from oracle.pdhg_port import KktPoint, Model, PdhgState

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import paper_2603_03150_b200 as eng

    return eng


def _rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(1.0, float(np.max(np.abs(b)))))


@pytest.fixture(scope="module")
def c4small():
    from paper_2603_03150_b200.instances import config4

    return config4(scale=0.02, seed=11)   # 100k x 200k, ~4M nnz, band +-1000


@pytest.fixture(scope="module")
def c2small():
    from paper_2603_03150_b200.instances import config2

    return config2(scale=0.02, seed=12)   # 10k x ~23k, heavy-tailed rows (up to 1000)


SCALED_LAYOUTS = {"default": {}, "rows": dict(row_order="length", sell="on", sell_sort="off")}
if EXPERIMENTAL_BUILD:
    SCALED_LAYOUTS["psr"] = dict(psr="on")
PSR_PARAMS = ["off", "on"] if EXPERIMENTAL_BUILD else ["off"]


@pytest.mark.parametrize("layout", sorted(SCALED_LAYOUTS))
def test_iterates_scaled_config4(eng, c4small, layout):
    """First 100 iterates (incl. the iteration-64 check/restart) to 1e-9."""
    from paper_2603_03150_b200 import _native as N

    T = eng.types()
    p = c4small
    psr = "on" if layout == "psr" else "off"
    if psr == "on":
        skip_unless_experimental("psr")
    opts = eng.GpuOptions(**SCALED_LAYOUTS[layout])
    rec = {}
    keep = {1, 2, 17, 63, 64, 65, 100}
    oracle.run_pdhg(Model(p.A, p.b, p.c), oracle.PdhgParams(eps_rel=1e-12, max_kkt_passes=100),
                    on_step=lambda st: rec.__setitem__(st.iterations, (st.x.copy(), st.y.copy(),
                                                                        st.avg_x.copy(), st.avg_y.copy()))
                    if st.iterations in keep else None)
    for k in sorted(keep):
        ce = 10**6 if k % 64 == 0 else 64
        eng.run_pdhg(p, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=k, check_every=ce), gpu=opts)
        dev = eng.device_lp(p, opts)
        if psr == "on":
            assert dev.psr_info["A"]["used"] and dev.psr_info["At"]["used"]
        if layout == "rows":
            assert dev.row_perm is not None and dev.sell_info["A"]["used"]
        x, y, _ = dev.fetch(N.PT_CUR, want_z=False)
        ax, ay, _ = dev.fetch(N.PT_AVG, want_z=False)
        ox, oy, oax, oay = rec[k]
        assert _rel(x, ox) <= 1e-9 and _rel(y, oy) <= 1e-9, k
        assert _rel(ax, oax) <= 1e-9 and _rel(ay, oay) <= 1e-9, k


@pytest.mark.skipif(not EXPERIMENTAL_BUILD, reason="PSR: experiment build only")
def test_psr_and_csr_agree_full_run(eng, c4small):
    """Both layouts reach 1e-4 with the same iteration count; the point passes KKT."""
    skip_unless_experimental("psr")
    T = eng.types()
    p = c4small
    runs = {}
    for psr in ("off", "on"):
        pt, st = eng.run_pdhg(p, T.PdhgParams(eps_rel=1e-4), gpu=eng.GpuOptions(psr=psr))
        assert st.status.value == "Optimal"
        t = oracle.check_relative_termination(Model(p.A, p.b, p.c), KktPoint(pt.x, pt.y, pt.z), 1e-4)
        assert t.ok
        runs[psr] = (st.iterations, float(p.c @ pt.x))
    assert abs(runs["on"][0] - runs["off"][0]) <= 0.05 * runs["off"][0]
    assert runs["on"][1] == pytest.approx(runs["off"][1], rel=1e-6)


@pytest.mark.parametrize("psr", PSR_PARAMS)
def test_heavy_rows_config2(eng, c2small, psr):
    """Heavy-tailed rows (block-per-row path) against the oracle, 100 iterates."""
    from paper_2603_03150_b200 import _native as N

    if psr == "on":
        skip_unless_experimental("psr")
    T = eng.types()
    p = c2small
    opts = eng.GpuOptions(psr=psr, heavy_threshold=128, psr_min_rows=1)
    dev = None
    st_o = {}
    oracle.run_pdhg(Model(p.A, p.b, p.c), oracle.PdhgParams(eps_rel=1e-12, max_kkt_passes=100),
                    on_step=lambda st: st_o.__setitem__(st.iterations, (st.x.copy(), st.y.copy()))
                    if st.iterations in (1, 50, 100) else None)
    for k in (1, 50, 100):
        eng.run_pdhg(p, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=k), gpu=opts)
        dev = eng.device_lp(p, opts)
        x, y, _ = dev.fetch(N.PT_CUR, want_z=False)
        assert _rel(x, st_o[k][0]) <= 1e-9 and _rel(y, st_o[k][1]) <= 1e-9, k
    assert dev._prob.a_n_heavy > 0


@pytest.mark.parametrize("layout", sorted(SCALED_LAYOUTS))
def test_spmv_scaled_1e12(eng, c4small, layout):
    p = c4small
    if layout == "psr":
        skip_unless_experimental("psr")
    dev = eng.device_lp(p, eng.GpuOptions(**SCALED_LAYOUTS[layout]))
    rng = np.random.default_rng(5)
    v = rng.standard_normal(p.n)
    w = rng.standard_normal(p.m)
    assert _rel(dev.spmv(v), p.A @ v) <= 1e-12
    assert _rel(dev.spmv(w, transpose=True), p.A.T @ w) <= 1e-12


# ---------------------------------------------------------------- full config-4 size
@pytest.fixture(scope="module")
def c4full():
    from paper_2603_03150_b200.instances import config4

    return config4(scale=1.0, seed=4)     # the bench instance: 5M x 10M, 199.9M nnz


def test_full_config4_spmv_1e12(eng, c4full):
    """Single SpMV gate (1e-12 relative) at the full 200M-nnz size, both operators."""
    p = c4full
    dev = eng.device_lp(p, eng.GpuOptions(cache_layout=False))
    rng = np.random.default_rng(9)
    v = rng.standard_normal(p.n)
    w = rng.standard_normal(p.m)
    assert _rel(dev.spmv(v), p.A @ v) <= 1e-12
    assert _rel(dev.spmv(w, transpose=True), p.A.T @ w) <= 1e-12


def test_full_config4_first_iterates_1e9(eng, c4full):
    """Iterates 1-2 at full size against the oracle's pdhg_step with the same step size."""
    from paper_2603_03150_b200 import _native as N

    T = eng.types()
    p = c4full
    lam = eng.estimate_opnorm(p.A)
    opts = eng.GpuOptions(opnorm=lam)
    step = 1.0 / (1.05 * lam)                                 # pdhg.py:119
    st = PdhgState(x=np.zeros(p.n), y=np.zeros(p.m), avg_x=np.zeros(p.n), avg_y=np.zeros(p.m),
                   avg_weight=0.0, tau=step, sigma=step, omega=1.0, iterations=0, restarts=0,
                   restart_x=None, restart_y=None, restart_score=1.0)
    model = Model(p.A, p.b, p.c)
    for k in (1, 2):
        oracle.pdhg_step(st, model)
        eng.run_pdhg(p, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=k, check_every=10**6), gpu=opts)
        dev = eng.device_lp(p, opts)
        x, y, _ = dev.fetch(N.PT_CUR, want_z=False)
        assert _rel(x, st.x) <= 1e-9 and _rel(y, st.y) <= 1e-9, k


def test_full_config4_reaches_1e4(eng, c4full):
    """Full run to 1e-4 at full size; the returned point re-passes the oracle's
    termination test (size-independent property; iteration count is a multiple
    of check_every)."""
    T = eng.types()
    p = c4full
    pt, st = eng.run_pdhg(p, T.PdhgParams(eps_rel=1e-4, time_limit_s=300))
    assert st.status.value == "Optimal"
    assert st.iterations % 64 == 0
    t = oracle.check_relative_termination(Model(p.A, p.b, p.c), KktPoint(pt.x, pt.y, pt.z), 1e-4)
    assert t.ok
    assert st.history and st.history[-1]["iteration"] == st.iterations
