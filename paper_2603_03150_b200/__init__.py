"""paper_2603_03150_b200 -- B200-native engine for the PDHG hot path of arxiv 2603.03150.

Drop-in replacement for the reference package's ``hybridlp.pdhg.run_pdhg``
(/root/reference/pkg/src/hybridlp/pdhg.py:162-258): the Python host keeps
the reference's signature, options, result objects and control flow, and
every arithmetic step runs in hand-written sm_100a CUDA kernels behind the
C ABI in include/pdhg_b200.h (libpdhg_b200.so).  There is no CPU fallback.

    from paper_2603_03150_b200 import run_pdhg, install
    install()          # rebind hybridlp's run_pdhg names to the GPU engine
"""

from __future__ import annotations

from .engine import DeviceLp, GpuOptions, clear_cache, device_lp, estimate_opnorm, run_pdhg
from .lp_types import resolve as types

__all__ = ["run_pdhg", "estimate_opnorm", "GpuOptions", "DeviceLp", "device_lp", "clear_cache",
           "install", "uninstall", "types"]

# the four modules that bind `run_pdhg` at import time:
# hybridlp/__init__.py:35, pdhg.py:162, warmstart.py:33, bench.py:24
_REBIND = ("hybridlp", "hybridlp.pdhg", "hybridlp.warmstart", "hybridlp.bench")
_saved: dict = {}


def install() -> None:
    """Route every ``run_pdhg`` name of the reference package to this engine."""
    import importlib

    for name in _REBIND:
        mod = importlib.import_module(name)
        if name not in _saved:
            _saved[name] = getattr(mod, "run_pdhg")
        setattr(mod, "run_pdhg", run_pdhg)


def uninstall() -> None:
    import importlib

    for name, fn in list(_saved.items()):
        setattr(importlib.import_module(name), "run_pdhg", fn)
        del _saved[name]
