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
from .ruiz import ruiz_equilibrate
from .stdform import to_standard_form

__all__ = ["run_pdhg", "estimate_opnorm", "ruiz_equilibrate", "to_standard_form", "GpuOptions",
           "DeviceLp", "device_lp", "clear_cache", "install", "uninstall", "types"]

# the four modules that bind `run_pdhg` at import time:
# hybridlp/__init__.py:35, pdhg.py:162, warmstart.py:33, bench.py:24
_REBIND = ("hybridlp", "hybridlp.pdhg", "hybridlp.warmstart", "hybridlp.bench")
_saved: dict = {}


# ruiz_equilibrate is bound in transform.py:35 and imported into warmstart.py:42
_REBIND_RUIZ = ("hybridlp", "hybridlp.transform", "hybridlp.warmstart")
# to_standard_form is bound in lp_core.py:250 (also called by
# evaluate_general_point, lp_core.py:490) and imported into warmstart.py:29
_REBIND_STD = ("hybridlp", "hybridlp.lp_core", "hybridlp.warmstart")


# centered_start is bound in warmstart.py:99 (called at 323) and re-exported in __init__.py:49
_REBIND_CENTER = ("hybridlp", "hybridlp.warmstart")


def install(ruiz: bool = False, std_form: bool = False, centered: bool = False) -> None:
    """Route every ``run_pdhg`` name of the reference package to this engine;
    with ``ruiz=True`` also its ``ruiz_equilibrate`` (device Ruiz, whose
    scaled matrix then stays on the device for the PDHG solve); with
    ``std_form=True`` also ``to_standard_form`` (device builder, whose
    matrix the device Ruiz then reuses); with ``centered=True`` also
    ``centered_start`` (the hand-off of the PDHG point to the IPM)."""
    import importlib

    targets = [(n, "run_pdhg", run_pdhg) for n in _REBIND]
    if ruiz:
        targets += [(n, "ruiz_equilibrate", ruiz_equilibrate) for n in _REBIND_RUIZ]
    if std_form:
        targets += [(n, "to_standard_form", to_standard_form) for n in _REBIND_STD]
    if centered:
        from .finish import centered_start

        targets += [(n, "centered_start", centered_start) for n in _REBIND_CENTER]
    for name, attr, fn in targets:
        mod = importlib.import_module(name)
        if (name, attr) not in _saved:
            _saved[(name, attr)] = getattr(mod, attr)
        setattr(mod, attr, fn)


def uninstall() -> None:
    import importlib

    for (name, attr), fn in list(_saved.items()):
        setattr(importlib.import_module(name), attr, fn)
        del _saved[(name, attr)]
