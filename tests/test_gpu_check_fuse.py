"""The two-point check's A side fused into the last iteration of a period
(GpuOptions.check_fuse, pdhg_check_fuse_enable).

At every check (pdhg.py:198-204) the reference scores the current and the
averaged point, i.e. computes A x and A avg_x (lp_core.py:436).  The engine
runs the period's last iteration with (xe, x, avg_x) quads: its dual step
(pdhg.py:143) gathers all three per entry and leaves each row's two primal
residuals, which the check accumulates in the separate A-side kernel's exact
order.  Every iterate, every check scalar and every decision must be bit for
bit those of the unfused path.
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
    "sell_rows_cols": dict(sell="on", row_order="length", row_order_window=64, col_order="length"),
}


@pytest.fixture(scope="module")
def eng():
    import paper_2603_03150_b200 as e

    return e


def _bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.uint64)


def _same(a, b):
    (pa, sa), (pb, sb) = a, b
    assert sa.status == sb.status and sa.iterations == sb.iterations and sa.restarts == sb.restarts
    for u, v in ((pa.x, pb.x), (pa.y, pb.y), (pa.z, pb.z)):
        assert np.array_equal(_bits(u), _bits(v))
    assert len(sa.history) == len(sb.history)
    for ha, hb in zip(sa.history, sb.history):
        for key in ("cur_max_violation", "avg_max_violation", "restart", "omega"):
            assert ha[key] == hb[key], key
        for key in ("cur_termination", "avg_termination"):
            ta, tb = ha[key], hb[key]
            for f in ("primal_lhs", "dual_lhs", "gap_lhs", "gap_rhs", "ok"):
                assert getattr(ta, f) == getattr(tb, f), (key, f)


class _Lp:
    """The (A, b, c) view run_pdhg takes of a generated instance."""

    def __init__(self, inst):
        self.A, self.b, self.c = inst.A, inst.b, inst.c


def _run(eng, p, params, on, **kw):
    opts = eng.GpuOptions(cache_layout=False, check_fuse=on, **kw)
    return eng.run_pdhg(p, params, gpu=opts)


@pytest.mark.parametrize("layout", sorted(SELL_LAYOUTS))
@pytest.mark.parametrize("name", GOLDEN_NAMES)
@pytest.mark.parametrize("eps,limit", [(1e-6, 200_000), (1e-12, 200)])
def test_check_fuse_is_bitwise_neutral(eng, name, layout, eps, limit):
    gm = load_golden(name)
    params = eng.types().PdhgParams(eps_rel=eps, max_kkt_passes=limit)
    _same(_run(eng, gm, params, True, **SELL_LAYOUTS[layout]),
          _run(eng, gm, params, False, **SELL_LAYOUTS[layout]))


@pytest.mark.parametrize("check_every", [1, 2, 3, 64])
def test_check_fuse_short_periods(eng, check_every):
    """check_every = 1: one-iteration periods (never fused: the last iteration
    is also the first); 2, 3: the fused iteration right after the check-dot
    first step; an iteration limit that is not a multiple of check_every."""
    gm = load_golden(GOLDEN_NAMES[0])
    params = eng.types().PdhgParams(eps_rel=1e-12, max_kkt_passes=100 + check_every,
                                    check_every=check_every)
    _same(_run(eng, gm, params, True, sell="on"), _run(eng, gm, params, False, sell="on"))


def test_check_fuse_scalars_through_the_abi(eng):
    """Raw scalars of run_period_check (all 16 of the two points) bitwise,
    fused and unfused contexts stepping the same iterates."""
    from paper_2603_03150_b200 import _native as N
    from paper_2603_03150_b200.engine import _start_vector

    gm = load_golden(GOLDEN_NAMES[-1])
    devs = [eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions(cache_layout=False, sell="on", check_fuse=on))
            for on in (True, False)]
    assert devs[0].check_fuse and not devs[1].check_fuse
    out = []
    for d in devs:
        lam = d.opnorm(_start_vector(d.n, 0))
        st = 1.0 / (1.05 * lam)
        d.reset()
        qs = []
        for r in range(4):
            fail, q = d.run_period_check(64, 64 * r, st, st, float(64 * r), N.PT_CUR, N.PT_AVG)
            assert fail < 0
            qs.append(np.asarray(q, dtype=np.float64).copy())
        x, y, z = d.fetch(N.PT_AVG)
        out.append((qs, x, y, z))
    for a, b in zip(out[0][0], out[1][0]):
        assert np.array_equal(_bits(a), _bits(b))
    for u, v in zip(out[0][1:], out[1][1:]):
        assert np.array_equal(_bits(u), _bits(v))


def test_check_fuse_heavy_rows(eng):
    """Config 2 at 0.2 % with a low heavy threshold: block-per-row rows of A
    take the fused dual step's block branch (row_dot order + block sums)."""
    from paper_2603_03150_b200.instances import config2

    inst = config2(0.002, seed=2)
    params = eng.types().PdhgParams(eps_rel=1e-12, max_kkt_passes=256)
    kw = dict(sell="on", heavy_threshold=64)
    d = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False, **kw))
    assert d.check_fuse and d.a_heavy.numel() > 0
    p = _Lp(inst)
    _same(_run(eng, p, params, True, **kw), _run(eng, p, params, False, **kw))


def test_check_fuse_scaled_config4(eng):
    """Config 4 at 2 % with the automatic renumbering and both sliced-ELL
    layouts: 640 iterations (10 checks) fused and unfused, bitwise."""
    from paper_2603_03150_b200.instances import config4

    p = _Lp(config4(0.02, seed=4))
    params = eng.types().PdhgParams(eps_rel=1e-12, max_kkt_passes=640)
    _same(_run(eng, p, params, True, sell="on"), _run(eng, p, params, False, sell="on"))


def test_check_fuse_enabled_only_where_it_applies(eng):
    gm = load_golden(GOLDEN_NAMES[0])
    assert eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions(cache_layout=False, sell="on")).check_fuse
    assert not eng.DeviceLp(gm.A, gm.b, gm.c, eng.GpuOptions(cache_layout=False, sell="off")).check_fuse
    assert not eng.DeviceLp(gm.A, gm.b, gm.c,
                            eng.GpuOptions(cache_layout=False, sell="on", check_fuse=False)).check_fuse


@pytest.mark.parametrize("check_every", [64, 5])
def test_check_fuse_numerical_failure(eng, check_every):
    """A model whose x overflows at iteration 335 (pdhg.py:194-196): inside a
    fused period (check_every 64) and in the fused last iteration itself
    (check_every 5: the period 331-335 ends there) -- the failure exit, its
    best point and z are bitwise those of the unfused path."""
    from test_sharded_cpu import failing_block_model

    p = failing_block_model()
    params = eng.types().PdhgParams(eps_rel=1e-6, max_kkt_passes=500, check_every=check_every)
    on = _run(eng, p, params, True, sell="on")
    off = _run(eng, p, params, False, sell="on")
    assert on[1].status.value == "NumericalFailure" and on[1].iterations == 335
    _same(on, off)
