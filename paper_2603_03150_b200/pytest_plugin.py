"""pytest plugin: run the reference package's own tests against the GPU engine.

    PYTHONPATH=oracle/_ref/site:. python -m pytest \
        -p paper_2603_03150_b200.pytest_plugin oracle/_ref/tests

(``oracle/make_ref.sh`` builds oracle/_ref from /root/reference/pkg; in the
build container ``/root/reference/pkg/{src,tests}`` work the same way.)

The rebinding happens in ``pytest_configure``, before test modules are
collected, because conftest.py:21-28, test_pdhg.py:7-20 and the other test
modules import the names at module load.  ``PDHG_B200_ROUTE`` picks what is
routed: ``pdhg`` (default) rebinds ``run_pdhg`` in the four modules that bind
it; ``all`` also routes ``ruiz_equilibrate``,
``to_standard_form`` and ``centered_start`` (the §8(f) rows) through
``install(ruiz=True, std_form=True, centered=True)``.  Every routed call is
counted, and the summary line proves the GPU path ran.
"""

from __future__ import annotations

import functools
import os

CALLS: dict = {}


def _counted(name, fn):
    CALLS.setdefault(name, 0)

    @functools.wraps(fn)
    def wrapper(*a, **k):
        CALLS[name] += 1
        return fn(*a, **k)

    return wrapper


def pytest_configure(config):
    import importlib

    from . import _native, engine, finish, ruiz, stdform

    _native.load()                      # fail loudly without the CUDA library
    route = os.environ.get("PDHG_B200_ROUTE", "pdhg")
    if route not in ("pdhg", "all"):
        raise ValueError(f"PDHG_B200_ROUTE must be 'pdhg' or 'all', not {route!r}")
    targets = [(m, "run_pdhg", engine.run_pdhg)
               for m in ("hybridlp", "hybridlp.pdhg", "hybridlp.warmstart", "hybridlp.bench")]
    if route == "all":
        targets += [(m, "ruiz_equilibrate", ruiz.ruiz_equilibrate)
                    for m in ("hybridlp", "hybridlp.transform", "hybridlp.warmstart")]
        targets += [(m, "to_standard_form", stdform.to_standard_form)
                    for m in ("hybridlp", "hybridlp.lp_core", "hybridlp.warmstart")]
        targets += [(m, "centered_start", finish.centered_start)
                    for m in ("hybridlp", "hybridlp.warmstart")]
    wrapped = {}
    for mod, attr, fn in targets:
        if attr not in wrapped:
            wrapped[attr] = _counted(attr, fn)
        setattr(importlib.import_module(mod), attr, wrapped[attr])


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"paper_2603_03150_b200: run_pdhg calls routed to GPU engine: "
                                f"{CALLS.get('run_pdhg', 0)}")
    for name in ("ruiz_equilibrate", "to_standard_form", "centered_start"):
        if name in CALLS:
            terminalreporter.write_line(f"paper_2603_03150_b200: {name} calls routed to GPU engine: "
                                        f"{CALLS[name]}")
