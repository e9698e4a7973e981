"""Re-entrancy (SURVEY §8(b) "Threading"): the reference's bench runs
run_pdhg from ThreadPoolExecutor workers on different models at once
(bench.py:415-420).  Concurrent calls -- different models, and the same model
twice -- return exactly what sequential calls return."""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import pytest

from conftest import GOLDEN_NAMES, load_golden

pytestmark = pytest.mark.gpu


def test_concurrent_run_pdhg_matches_sequential():
    import paper_2603_03150_b200 as eng

    T = eng.types()
    names = list(GOLDEN_NAMES)[:6]
    models = [load_golden(nm) for nm in names]
    jobs = models + models[:2]           # two models run twice, concurrently
    params = T.PdhgParams(eps_rel=1e-6, max_kkt_passes=5_000)
    eng.clear_cache()
    seq = [eng.run_pdhg(gm, params) for gm in jobs]
    eng.clear_cache()
    with ThreadPoolExecutor(4) as ex:
        par = list(ex.map(lambda gm: eng.run_pdhg(gm, params), jobs))
    for (ps, ss), (pp, sp_) in zip(seq, par):
        assert (ss.status, ss.iterations, ss.restarts) == (sp_.status, sp_.iterations, sp_.restarts)
        assert ps.x.tobytes() == pp.x.tobytes() and ps.y.tobytes() == pp.y.tobytes()
        assert ps.z.tobytes() == pp.z.tobytes()


def test_concurrent_ruiz_and_stdform():
    """The §8(f) device rows from several threads (separate streams, shared staging ring)."""
    import numpy as np

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.instances import config4

    insts = [config4(scale=0.02, seed=s) for s in range(4)]
    seq = [eng.ruiz_equilibrate(p, register_layout=False) for p in insts]
    with ThreadPoolExecutor(4) as ex:
        par = list(ex.map(lambda p: eng.ruiz_equilibrate(p, register_layout=False), insts))
    for (s1, i1), (s2, i2) in zip(seq, par):
        assert s1.A.data.tobytes() == s2.A.data.tobytes()
        assert np.array_equal(i1.row_scale, i2.row_scale) and np.array_equal(i1.col_scale, i2.col_scale)
