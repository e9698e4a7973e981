"""GPU parity: the sm_100a path vs the reference (golden files) and the CPU oracle.

Gates (BASELINE.json north_star):
  * a single SpMV agrees to 1e-12 relative;
  * the first 100 iterates agree to 1e-9 relative (this includes the
    check -> candidate -> restart -> omega logic at iteration 64);
  * full runs: same status, iteration count exactly equal (checks happen
    every 64 iterations, so +-5% means equal below 1,280), objective within
    1e-6 relative, and the returned point meets all three KKT criteria.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import EXPERIMENTAL_BUILD, GOLDEN_NAMES, load_golden

pytestmark = pytest.mark.gpu

SPMV_RTOL = 1e-12
ITER_RTOL = 1e-9


@pytest.fixture(scope="module")
def eng():
    import paper_2603_03150_b200 as eng

    return eng


# the step kernels' layouts: CSR-vector (also split-K), sliced ELL, and PSR
# with every entry staged in shared-memory panels or gathered from global memory
LAYOUTS = {
    "csr": dict(psr="off", sell="off", persistent="off"),
    "sell": dict(psr="off", sell="on", sell_sort="off", persistent="off"),
    "sell_sorted": dict(psr="off", sell="on", sell_sort="on", persistent="off"),
    # constraints renumbered by length inside windows of 64 rows (row_order),
    # sliced ELL on the renumbered A; y mapped back on download
    "sell_rows": dict(psr="off", sell="on", sell_sort="off", persistent="off", row_order="length",
                      row_order_window=64),
    "persistent": dict(psr="off", sell="off", persistent="on"),
    "tiny": dict(psr="off", sell="off", persistent="tiny"),
    "csr_split2": dict(psr="off", sell="off", persistent="off", dual_split=2),
    # every row longer than its lane count runs warp-per-row (the medium tier)
    "csr_medium": dict(psr="off", sell="off", persistent="off", medium_per_lane=1),
    "psr_staged": dict(psr="on", psr_min_staged=1),
    "psr_remote": dict(psr="on", psr_min_staged=10**9),
}


# layouts compiled only into the experiment build (measured slower):
# parametrized only when that build is loaded
EXPERIMENTAL = {"persistent", "tiny", "psr_staged", "psr_remote"}
LAYOUT_NAMES = sorted(k for k in LAYOUTS if EXPERIMENTAL_BUILD or k not in EXPERIMENTAL)


def _opts(eng, layout):
    if layout in EXPERIMENTAL:
        from paper_2603_03150_b200 import _native

        if not _native.experimental():
            pytest.skip(f"{layout}: experiment build only (PDHG_B200_LIB=tools/_libs/libpdhg_b200_exp.so)")
    return eng.GpuOptions(**LAYOUTS[layout])


def _rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_single_spmv_1e12(eng, name):
    gm = load_golden(name)
    dev = eng.device_lp(gm, eng.GpuOptions())
    Av = dev.spmv(gm.g["spmv_v"], transpose=False)
    Atw = dev.spmv(gm.g["spmv_w"], transpose=True)
    assert _rel(Av, gm.g["spmv_Av"]) <= SPMV_RTOL
    assert _rel(Atw, gm.g["spmv_Atw"]) <= SPMV_RTOL


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_opnorm_matches_reference(eng, name):
    gm = load_golden(name)
    lam = eng.estimate_opnorm(gm.A, seed=0)
    assert lam == pytest.approx(float(gm.g["opnorm_seed0"]), rel=1e-12)


@pytest.mark.parametrize("layout", LAYOUT_NAMES)
@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_first_100_iterates_1e9(eng, name, layout):
    """Run k iterations on the GPU for each captured k and compare the state.

    max_kkt_passes=k with eps=1e-12 stops right after step k; the returned
    best point is not the iterate, so read the device state directly.
    """
    gm = load_golden(name)
    g = gm.g
    from paper_2603_03150_b200 import _native as N

    for j, k in enumerate(g["it_k"]):
        k = int(k)
        if j % 3 and k not in (63, 64, 65, 100):
            continue
        # a check at k itself would already have restarted; the reference
        # capture is taken right after the step (before the check)
        ce = 10**6 if k % 64 == 0 else 64
        opts = _opts(eng, layout)
        eng.run_pdhg(gm, _params(eng, eps_rel=1e-12, max_kkt_passes=k, check_every=ce), gpu=opts)
        dev = eng.device_lp(gm, opts)
        if layout.startswith("psr"):
            assert dev.psr_info["A"].get("used") and dev.psr_info["At"].get("used")
        if layout == "csr_split2" and gm.n >= 8:
            assert dev.nsplit == 2
        x, y, _ = dev.fetch(N.PT_CUR, want_z=False)
        ax, ay, _ = dev.fetch(N.PT_AVG, want_z=False)
        assert _rel(x, g["it_x"][j]) <= ITER_RTOL, (name, k)
        assert _rel(y, g["it_y"][j]) <= ITER_RTOL, (name, k)
        assert _rel(ax, g["it_avgx"][j]) <= ITER_RTOL, (name, k)
        assert _rel(ay, g["it_avgy"][j]) <= ITER_RTOL, (name, k)


def _params(eng, **kw):
    return eng.types().PdhgParams(**kw)


@pytest.mark.parametrize("layout", LAYOUT_NAMES)
@pytest.mark.parametrize("name", GOLDEN_NAMES)
@pytest.mark.parametrize("tag,eps,limit", [("e4", 1e-4, 200_000), ("e6", 1e-6, 200_000),
                                           ("lim128", 1e-12, 128), ("lim200", 1e-12, 200)])
def test_full_run_parity(eng, name, tag, eps, limit, layout):
    gm = load_golden(name)
    r = gm.run(tag)
    pt, st = eng.run_pdhg(gm, _params(eng, eps_rel=eps, max_kkt_passes=limit), gpu=_opts(eng, layout))
    assert st.status.value == str(r["status"])
    ref_it = int(r["iterations"])
    if ref_it < 1280:
        assert st.iterations == ref_it
    else:
        assert abs(st.iterations - ref_it) <= 0.05 * ref_it
    assert st.restarts == int(r["restarts"]) or ref_it >= 1280
    obj = float(gm.c @ pt.x)
    assert obj == pytest.approx(float(r["obj"]), rel=1e-6, abs=1e-9)
    if str(r["status"]) == "Optimal":
        assert st.termination.ok
        # post-hoc: the returned point re-passes the relative check (oracle)
        import oracle
        from oracle.pdhg_port import KktPoint, Model

        t = oracle.check_relative_termination(Model(gm.A, gm.b, gm.c), KktPoint(pt.x, pt.y, pt.z), eps)
        assert t.ok
    else:
        np.testing.assert_allclose(pt.x, r["x"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(pt.y, r["y"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(pt.z, r["z"], rtol=1e-9, atol=1e-12)
        ref_t = r["term"]
        t = st.termination
        got = np.array([t.primal_lhs, t.primal_rhs, t.dual_lhs, t.dual_rhs, t.gap_lhs, t.gap_rhs])
        np.testing.assert_allclose(got, ref_t, rtol=1e-9, atol=1e-14)


@pytest.mark.parametrize("layout", LAYOUT_NAMES)
def test_deterministic_bitwise(eng, layout):
    gm = load_golden("config0_s0")
    eng.clear_cache()
    pt1, s1 = eng.run_pdhg(gm, _params(eng, eps_rel=1e-4), seed=3, gpu=_opts(eng, layout))
    eng.clear_cache()
    pt2, s2 = eng.run_pdhg(gm, _params(eng, eps_rel=1e-4), seed=3, gpu=_opts(eng, layout))
    np.testing.assert_array_equal(pt1.x, pt2.x)
    np.testing.assert_array_equal(pt1.y, pt2.y)
    assert s1.iterations == s2.iterations


def test_time_limit_zero(eng):
    gm = load_golden("lp2_ruiz")
    pt, st = eng.run_pdhg(gm, _params(eng, eps_rel=1e-4, time_limit_s=0.0))
    assert st.status.value == "TimeLimit"
    assert st.iterations == 0
    assert pt.x.size == gm.n


def test_history_field(eng):
    gm = load_golden("eq_20x35_s17_ruiz")
    pt, st = eng.run_pdhg(gm, _params(eng, eps_rel=1e-6))
    assert len(st.history) == st.iterations // 64
    assert sum(h["restart"] for h in st.history) == st.restarts
    assert st.history[-1]["iteration"] == st.iterations
