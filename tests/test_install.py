"""install() rebinds the reference's run_pdhg names (needs the reference
package importable: /root/reference in the build container)."""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")


@pytest.fixture
def hybridlp():
    if not REF.exists():
        pytest.skip("reference tree not available")
    sys.path.insert(0, str(REF))
    import hybridlp

    from paper_2603_03150_b200 import lp_types

    lp_types.reset_cache()
    yield hybridlp
    sys.path.remove(str(REF))
    lp_types.reset_cache()


def test_install_rebinds_all_four_names(hybridlp):
    import importlib

    import paper_2603_03150_b200 as eng

    mods = ["hybridlp", "hybridlp.pdhg", "hybridlp.warmstart", "hybridlp.bench"]
    before = {m: importlib.import_module(m).run_pdhg for m in mods}
    eng.install(ruiz=True)
    try:
        for m in mods:
            assert importlib.import_module(m).run_pdhg is eng.run_pdhg
        for m in ("hybridlp", "hybridlp.transform", "hybridlp.warmstart"):
            assert importlib.import_module(m).ruiz_equilibrate is eng.ruiz_equilibrate
    finally:
        eng.uninstall()
    for m in mods:
        assert importlib.import_module(m).run_pdhg is before[m]


def test_result_types_are_the_references(hybridlp):
    from paper_2603_03150_b200.lp_types import resolve

    T = resolve()
    assert T.reference
    assert T.KktPoint is hybridlp.KktPoint
    assert T.PdhgParams is hybridlp.PdhgParams
    assert issubclass(T.SolveStats, hybridlp.SolveStats)
    st = T.SolveStats(status=hybridlp.SolveStatus.OPTIMAL, iterations=1, restarts=0,
                      wall_seconds=0.0, termination=None, max_violation=0.0)
    assert st.history == []


def test_install_rebinds_std_form_and_centering(hybridlp):
    import importlib

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200 import finish

    eng.install(std_form=True, centered=True)
    try:
        for m in ("hybridlp", "hybridlp.lp_core", "hybridlp.warmstart"):
            assert importlib.import_module(m).to_standard_form is eng.to_standard_form
        for m in ("hybridlp", "hybridlp.warmstart"):
            assert importlib.import_module(m).centered_start is finish.centered_start
    finally:
        eng.uninstall()
    assert importlib.import_module("hybridlp.warmstart").centered_start is not finish.centered_start
