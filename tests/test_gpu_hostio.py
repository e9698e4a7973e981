"""Chunked pinned-ring transfers (paper_2603_03150_b200/hostio.py): byte-exact
round trips across chunk boundaries, dtype casts on upload, concurrent callers."""

from __future__ import annotations

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("count,dtype", [(10, np.float64), (3_000_001, np.float64),
                                         (9_000_017, np.int32), (40_000_003, np.int8),
                                         (4 * (64 << 20) // 8 + 5, np.float64)])
def test_round_trip_bit_exact(count, dtype):
    import torch

    from paper_2603_03150_b200 import hostio

    rng = np.random.default_rng(count)
    a = rng.integers(-100, 100, size=count).astype(dtype)
    if dtype == np.float64:
        a = rng.standard_normal(count)
        a[::7] = np.nan
    d = hostio.h2d(a, dtype, "cuda")
    assert d.device.type == "cuda" and d.numel() == count
    torch.cuda.synchronize()
    back = hostio.d2h(d)
    assert back.dtype == a.dtype and back.tobytes() == a.tobytes()


def test_upload_casts_like_numpy():
    from paper_2603_03150_b200 import hostio

    a = np.arange(5_000_000, dtype=np.int64)
    d = hostio.h2d(a, np.int32, "cuda")
    assert hostio.d2h(d).tobytes() == a.astype(np.int32).tobytes()


def test_concurrent_callers():
    import torch

    from paper_2603_03150_b200 import hostio

    arrs = [np.random.default_rng(s).standard_normal(6_000_000 + s) for s in range(4)]
    out = [None] * 4

    def work(i):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            d = hostio.h2d(arrs[i], np.float64, "cuda")
            out[i] = hostio.d2h(d * 2.0)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(4):
        assert out[i].tobytes() == (arrs[i] * 2.0).tobytes()
