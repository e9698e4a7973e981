"""Host <-> device transfers of the large model arrays (matrix, vectors).

The public API takes and returns pageable numpy arrays (StandardLp, KktPoint),
and a plain ``torch.from_numpy(a).to(dev)`` of pageable memory runs at
~10 GB/s: the driver stages it through its own small pinned buffer with one
CPU thread.  Here a ring of pinned chunks is filled by several host threads
(numpy copies release the GIL) while the DMA engine drains the previous
chunks, so the host copy, the first-touch page faults of fresh destination
arrays and the PCIe transfer overlap.  Byte-for-byte copies: no conversion
happens on the way (dtype casts are done by numpy before the upload).

The staging ring is allocated once per device and process and guarded by a
lock (run_pdhg may be called from several threads, bench.py:415-420 of the
reference).
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

CHUNK = 64 << 20          # bytes per staging buffer (tools/hostio_lab.py: 64 MB x 4, 8-16 threads)
NBUF = 4                  # buffers in the ring
SMALL = 8 << 20           # below this, the plain torch copy
PIECE = 4 << 20           # host-copy granularity per thread

_pool = None
_pool_lock = threading.Lock()
_rings: dict = {}


def _threads() -> int:
    return max(1, min(16, os.cpu_count() or 1))


def _executor():
    global _pool
    with _pool_lock:
        if _pool is None:
            _pool = ThreadPoolExecutor(_threads(), thread_name_prefix="pdhg-hostio")
        return _pool


def submit(fn, *args):
    """Run fn(*args) on the host thread pool, overlapped with device work
    (e.g. the power iteration's start vector during the model upload);
    returns a concurrent.futures.Future."""
    return _executor().submit(fn, *args)


class _Ring:
    def __init__(self, dev):
        import torch

        self.lock = threading.Lock()
        self.bufs = [torch.empty(CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(NBUF)]
        self.np = [b.numpy() for b in self.bufs]
        self.events = [torch.cuda.Event() for _ in range(NBUF)]
        self.used = [False] * NBUF


def _ring(dev):
    import torch

    dev = torch.device(dev)
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    with _pool_lock:
        r = _rings.get(key)
        if r is None:
            with torch.cuda.device(key):
                r = _rings[key] = _Ring(key)
        return r


def _par_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src (flat uint8 views) split across the host threads."""
    n = src.size
    if n <= PIECE:
        np.copyto(dst, src)
        return
    k = min(_threads(), (n + PIECE - 1) // PIECE)
    step = (n + k - 1) // k
    futs = [_executor().submit(np.copyto, dst[o:o + step], src[o:o + step]) for o in range(0, n, step)]
    for f in futs:
        f.result()


def _flat_u8(a: np.ndarray) -> np.ndarray:
    return a.reshape(-1).view(np.uint8)


def h2d(a, dtype, dev):
    """Device copy of host array ``a`` (cast to ``dtype`` by numpy first), queued
    on the current stream of ``dev``; the caller orders later work on that stream."""
    import torch

    a = np.ascontiguousarray(a, dtype=dtype)
    if a.nbytes < SMALL:
        return torch.from_numpy(a).to(dev)
    out = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device=dev)
    src = _flat_u8(a)
    dst = out.view(-1).view(torch.uint8)
    r = _ring(dev)
    stream = torch.cuda.current_stream(dev)
    with r.lock:
        for i, off in enumerate(range(0, src.size, CHUNK)):
            k = i % NBUF
            if r.used[k]:
                r.events[k].synchronize()          # the DMA reading this buffer is done
            L = min(CHUNK, src.size - off)
            _par_copy(r.np[k][:L], src[off:off + L])
            dst[off:off + L].copy_(r.bufs[k][:L], non_blocking=True)
            r.events[k].record(stream)
            r.used[k] = True
        # the ring may be refilled by the next call only after these copies
        # have read it: that call synchronises on the same events
    return out


def d2h(t) -> np.ndarray:
    """Host numpy copy of contiguous device tensor ``t`` (queued behind the
    current stream's work on t's device; returns when the data is on the host)."""
    import torch

    t = t.contiguous()
    nbytes = t.numel() * t.element_size()
    if nbytes < SMALL:
        return t.cpu().numpy()
    out = np.empty(tuple(t.shape), dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    dst = _flat_u8(out)
    src = t.view(-1).view(torch.uint8)
    r = _ring(t.device)
    stream = torch.cuda.current_stream(t.device)
    pending = []
    with r.lock:
        def drain():
            k, off, L = pending.pop(0)
            r.events[k].synchronize()
            _par_copy(dst[off:off + L], r.np[k][:L])

        for i, off in enumerate(range(0, nbytes, CHUNK)):
            k = i % NBUF
            if len(pending) == NBUF:
                drain()
            elif r.used[k]:
                r.events[k].synchronize()          # an earlier call's DMA into this buffer
            L = min(CHUNK, nbytes - off)
            r.bufs[k][:L].copy_(src[off:off + L], non_blocking=True)
            r.events[k].record(stream)
            r.used[k] = True
            pending.append((k, off, L))
        while pending:
            drain()
    return out
