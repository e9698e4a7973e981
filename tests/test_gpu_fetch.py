"""pdhg_point_device + the pinned-ring download (DeviceLp.fetch) return
exactly what the synchronous pdhg_fetch copies."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("spec_name", ["PT_CUR", "PT_AVG", "PT_BEST"])
def test_point_device_matches_fetch(spec_name):
    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200 import _native as N
    from paper_2603_03150_b200.instances import config4

    p = config4(scale=0.01, seed=5)     # 2M entries: the ring path (> 8 MB vectors)
    dev = eng.DeviceLp(p.A, p.b, p.c, eng.GpuOptions(cache_layout=False))
    dev.reset()
    dev.run_period(64, 0, 1e-2, 1e-2, 0.0)
    dev.save_best(N.PT_AVG, N.BEST_XY | N.BEST_Z)
    dev.run_period(64, 64, 1e-2, 1e-2, 64.0)
    spec = getattr(N, spec_name)
    x, y, z = dev.fetch(spec)
    xr, yr, zr = np.empty(dev.n_full), np.empty(dev.m_full), np.empty(dev.n_full)
    N.check(dev.lib.pdhg_fetch(dev.ctx, spec, xr.ctypes.data, yr.ctypes.data, zr.ctypes.data))
    assert x.tobytes() == xr.tobytes() and y.tobytes() == yr.tobytes() and z.tobytes() == zr.tobytes()
    if spec == N.PT_BEST:
        x2, y2, z2 = dev.fetch(spec | N.SPEC_BEST_Z)
        N.check(dev.lib.pdhg_fetch(dev.ctx, spec | N.SPEC_BEST_Z, xr.ctypes.data, yr.ctypes.data,
                                   zr.ctypes.data))
        assert z2.tobytes() == zr.tobytes()
