"""Per-device pool of CUDA streams for the engine's contexts and one-shot steps.

torch's caching allocator keeps a freed block for reuse by allocations on the
stream it was allocated on.  A fresh stream per solve therefore never sees the
previous solve's freed blocks: every run_pdhg call cudaMalloc'ed its layout
anew (23 new segments, +16 GB reserved per config-4 call, and the upload /
layout timings of the e2e leg varied by 0.2-1.2 s; profiles/r02_setup_profile.log).
Streams taken from this pool return to it when their user is done, so the
next user on that device reuses both the stream and its cached blocks.
Concurrent users (threads) each hold a different stream.
"""

from __future__ import annotations

import threading

_lock = threading.Lock()
_free: dict[int, list] = {}


def acquire(dev):
    """A stream on ``dev`` (torch.device or index) no other pool user holds."""
    import torch

    idx = dev.index if isinstance(dev, torch.device) else int(dev)
    with _lock:
        pool = _free.setdefault(idx, [])
        if pool:
            return pool.pop()
    return torch.cuda.Stream(torch.device("cuda", idx))


def release(stream) -> None:
    """Give ``stream`` back (its queued work keeps its order; later users run after it)."""
    if stream is None:
        return
    with _lock:
        _free.setdefault(stream.device.index, []).append(stream)


class Borrowed:
    """``with Borrowed(dev) as s:`` -- a pooled stream for one call."""

    def __init__(self, dev):
        self.dev = dev
        self.stream = None

    def __enter__(self):
        self.stream = acquire(self.dev)
        return self.stream

    def __exit__(self, *exc):
        release(self.stream)
        return False
