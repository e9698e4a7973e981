"""The check -> next primal step reuse (GpuOptions.check_dot, pdhg_use_check_dot).

A two-point check computes A'y of the current and the averaged point
(pdhg.py:201-204 -> lp_core.py:437); the first primal step after it needs
A'y of the iterate it starts from (pdhg.py:142), which is one of those two
(the current point, or the average after a restart to it, pdhg.py:234-240).
The engine reuses the check's value; the check's dual side runs the primal
step's own row loop, so every iterate must be bit for bit the one computed
without the reuse.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN_NAMES, load_golden

pytestmark = pytest.mark.gpu

SELL_LAYOUTS = {
    "sell": dict(sell="on", sell_sort="off"),
    "sell_sorted": dict(sell="on", sell_sort="on"),
    "sell_rows": dict(sell="on", sell_sort="off", row_order="length", row_order_window=64),
}


@pytest.fixture(scope="module")
def eng():
    import paper_2603_03150_b200 as e

    return e


def _run(eng, p, params, layout, on):
    opts = eng.GpuOptions(cache_layout=False, check_dot=on, **SELL_LAYOUTS[layout])
    pt, st = eng.run_pdhg(p, params, gpu=opts)
    return pt, st


def _same(a, b):
    (pa, sa), (pb, sb) = a, b
    assert sa.status == sb.status and sa.iterations == sb.iterations and sa.restarts == sb.restarts
    for u, v in ((pa.x, pb.x), (pa.y, pb.y), (pa.z, pb.z)):
        assert np.array_equal(np.asarray(u).view(np.uint64), np.asarray(v).view(np.uint64))
    assert len(sa.history) == len(sb.history)
    for ha, hb in zip(sa.history, sb.history):
        assert ha["cur_max_violation"] == hb["cur_max_violation"]
        assert ha["avg_max_violation"] == hb["avg_max_violation"]
        assert ha["restart"] == hb["restart"]


_restart_kinds = set()


@pytest.mark.parametrize("layout", sorted(SELL_LAYOUTS))
@pytest.mark.parametrize("name", GOLDEN_NAMES)
@pytest.mark.parametrize("eps,limit", [(1e-6, 200_000), (1e-12, 200)])
def test_check_dot_is_bitwise_neutral(eng, name, layout, eps, limit):
    gm = load_golden(name)
    params = eng.types().PdhgParams(eps_rel=eps, max_kkt_passes=limit)
    on = _run(eng, gm, params, layout, True)
    off = _run(eng, gm, params, layout, False)
    _same(on, off)
    for h in on[1].history:
        if h["restart"]:
            _restart_kinds.add("avg" if h["avg_max_violation"] < h["cur_max_violation"] else "cur")


def test_both_restart_kinds_were_exercised():
    """Runs above restart both to the current point (slot 0) and to the
    average (slot 1), so both reuse slots were compared."""
    if not _restart_kinds:
        pytest.skip("run with the parametrized cases above")
    assert _restart_kinds == {"avg", "cur"}, _restart_kinds


def test_check_dot_enabled_only_where_it_applies(eng):
    gm = load_golden(GOLDEN_NAMES[0])
    d = eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions(cache_layout=False, sell="on"))
    assert d.check_dot
    d = eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions(cache_layout=False, sell="off"))
    assert not d.check_dot
    d = eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions(cache_layout=False, sell="on", check_dot=False))
    assert not d.check_dot


def test_use_check_dot_needs_a_two_point_check(eng):
    from paper_2603_03150_b200 import _native as N

    gm = load_golden(GOLDEN_NAMES[0])
    d = eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions(cache_layout=False, sell="on"))
    d.reset()
    with pytest.raises(N.NativeError):
        d.use_check_dot(0)                      # no check yet
    d.check(N.PT_CUR)
    with pytest.raises(N.NativeError):
        d.use_check_dot(0)                      # one-point check: no dots
    d.check(N.PT_CUR, N.PT_AVG)
    d.use_check_dot(1)                          # fine right after a two-point check
    d.run_period(64, 0, 0.1, 0.1, 0.0)          # consumes it
    with pytest.raises(N.NativeError):
        d.use_check_dot(0)


def test_check_dot_scaled_config4(eng):
    """Config 4 at 2 % (sliced ELL of A' forced: at 4M entries the automatic
    choice keeps CSR; renumbered A): 640 iterations (10 checks) with and
    without the reuse, bitwise."""
    from paper_2603_03150_b200.instances import config4

    inst = config4(0.02, seed=4)

    class P:
        pass

    p = P()
    p.A, p.b, p.c = inst.A, inst.b, inst.c
    params = eng.types().PdhgParams(eps_rel=1e-12, max_kkt_passes=640)
    res = []
    for on in (True, False):
        opts = eng.GpuOptions(cache_layout=False, check_dot=on, sell="on")
        res.append(eng.run_pdhg(p, params, gpu=opts))
    _same(res[0], res[1])
    assert eng.DeviceLp(p.A, p.b, p.c, eng.GpuOptions(cache_layout=False, sell="on")).check_dot


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_column_renumbering_maps_results_back(eng, name):
    """GpuOptions.col_order: the variables are relabelled on the device and
    x / z mapped back on download -- the run matches the unrenumbered one
    (same sums per row; only x-space reductions change order) and the single
    SpMV gate holds through the relabelling."""
    gm = load_golden(name)
    params = eng.types().PdhgParams(eps_rel=1e-12, max_kkt_passes=200)
    base = dict(cache_layout=False, sell="on", row_order="length", row_order_window=64)
    (pa, sa) = eng.run_pdhg(gm, params, gpu=eng.GpuOptions(col_order="length", **base))
    (pb, sb) = eng.run_pdhg(gm, params, gpu=eng.GpuOptions(col_order="natural", **base))
    assert sa.iterations == sb.iterations and sa.restarts == sb.restarts
    for u, v in ((pa.x, pb.x), (pa.y, pb.y), (pa.z, pb.z)):
        u, v = np.asarray(u), np.asarray(v)
        assert np.max(np.abs(u - v)) <= 1e-12 * max(1.0, float(np.max(np.abs(v))))
    d = eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions(col_order="length", **base))
    assert d.col_perm is not None
    v = gm.g["spmv_v"]
    w = gm.g["spmv_w"]
    assert np.max(np.abs(d.spmv(v) - gm.g["spmv_Av"])) <= 1e-12 * max(1.0, np.max(np.abs(gm.g["spmv_Av"])))
    assert np.max(np.abs(d.spmv(w, transpose=True) - gm.g["spmv_Atw"])) <= 1e-12 * max(
        1.0, np.max(np.abs(gm.g["spmv_Atw"])))
    from paper_2603_03150_b200.engine import _start_vector

    lam = d.opnorm(_start_vector(d.n, 0))          # start vector permuted on the device
    assert abs(lam - float(gm.g["opnorm_seed0"])) <= 1e-12 * float(gm.g["opnorm_seed0"])
