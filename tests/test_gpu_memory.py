"""Repeated solves reuse device memory (paper_2603_03150_b200/streams.py).

torch's caching allocator hands a freed block only to later allocations on
the stream it was allocated on; with a fresh stream per solve every call
cudaMalloc'ed its layout again and the reserved pool grew by the whole
layout per call.  Contexts now take their streams from a per-device pool.
"""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


def test_repeated_solves_allocate_no_new_segments():
    import torch

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.instances import config4

    inst = config4(0.02, seed=4)
    T = eng.types()
    params = T.PdhgParams(eps_rel=1e-12, max_kkt_passes=64)
    opts = eng.GpuOptions(cache_layout=False)
    eng.run_pdhg(inst, params, gpu=opts)          # first call: fills the allocator's pool
    torch.cuda.synchronize()
    stats = []
    for _ in range(3):
        s0 = torch.cuda.memory_stats()
        eng.run_pdhg(inst, params, gpu=opts)
        torch.cuda.synchronize()
        s1 = torch.cuda.memory_stats()
        stats.append((s1["segment.all.allocated"] - s0["segment.all.allocated"],
                      s1["reserved_bytes.all.current"] - s0["reserved_bytes.all.current"]))
    assert all(seg == 0 and grown <= 0 for seg, grown in stats), stats


def test_concurrent_contexts_hold_distinct_streams():
    from paper_2603_03150_b200 import streams

    import torch

    a = streams.acquire(0)
    b = streams.acquire(0)
    assert a.cuda_stream != b.cuda_stream
    streams.release(a)
    c = streams.acquire(0)
    assert c.cuda_stream == a.cuda_stream          # the pool hands the freed one back
    streams.release(b)
    streams.release(c)
    assert torch.cuda.is_available()
