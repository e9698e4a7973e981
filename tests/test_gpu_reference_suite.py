"""The reference package's OWN test suite, run against the GPU engine.

``oracle/make_ref.sh`` (build container) installs the unmodified reference
package into oracle/_ref/site and copies its tests to oracle/_ref/tests; the
directory is git-ignored but travels to the GPU box with the snapshot.  Each
case here runs that suite in a subprocess through
``paper_2603_03150_b200.pytest_plugin``, which rebinds the reference's
``run_pdhg`` names (and, with PDHG_B200_ROUTE=all, ``ruiz_equilibrate``,
``to_standard_form`` and ``centered_start``) to the CUDA engine before
collection, and asserts that every test passes and that the engine was
really called (/root/reference/pkg/tests/conftest.py:81-100,
test_pdhg.py:7-21,145-210, test_warmstart.py:154-211, test_bench.py:161-167,
192-201, test_acceptance.py:115-138).
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"


def _run_suite(route: str, files: list[str], timeout: int = 1800):
    if not (REF / "site" / "hybridlp").is_dir() or not (REF / "tests").is_dir():
        pytest.skip("oracle/_ref not built (bash oracle/make_ref.sh in the build container)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF / "site"), str(ROOT)])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env["PDHG_B200_ROUTE"] = route
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p",
           "paper_2603_03150_b200.pytest_plugin", "--rootdir", str(REF / "tests"),
           *([str(REF / "tests" / f) for f in files] or [str(REF / "tests")])]
    res = subprocess.run(cmd, env=env, cwd=str(REF / "tests"), capture_output=True, text=True,
                         timeout=timeout)
    out = res.stdout + res.stderr
    out_dir = ROOT / "gpurun_out"
    if out_dir.is_dir():
        (out_dir / f"reference_suite_{route}.log").write_text(out)
    calls = {k: int(v) for k, v in re.findall(r"(\w+) calls routed to GPU engine: (\d+)", out)}
    m = re.search(r"(\d+) passed", out)
    passed = int(m.group(1)) if m else 0
    assert res.returncode == 0, out[-6000:]
    assert not re.search(r"\d+ (failed|error)", out), out[-6000:]
    return passed, calls


PDHG_CONSUMERS = ["test_pdhg.py", "test_warmstart.py", "test_bench.py", "test_acceptance.py"]
# run_pdhg calls the unmodified reference suite makes (counted in the build
# container with a counting wrapper around the reference's own run_pdhg and no
# GPU: 34 over all 230 tests, all of them from these four files + conftest.py)
REFERENCE_RUN_PDHG_CALLS = 34


def test_reference_pdhg_consumers_route_to_gpu():
    """test_pdhg.py, test_warmstart.py, test_bench.py, test_acceptance.py with
    run_pdhg rebound: every test passes and every one of the suite's solves
    ran on the GPU."""
    passed, calls = _run_suite("pdhg", PDHG_CONSUMERS)
    assert passed >= 80, passed
    assert calls.get("run_pdhg", 0) == REFERENCE_RUN_PDHG_CALLS, calls


def test_reference_full_suite_all_rows_on_gpu():
    """The whole reference suite with run_pdhg, ruiz_equilibrate,
    to_standard_form and centered_start all routed to the device."""
    passed, calls = _run_suite("all", [])
    assert passed >= 230, passed
    assert calls.get("run_pdhg", 0) == REFERENCE_RUN_PDHG_CALLS, calls
    for name in ("ruiz_equilibrate", "to_standard_form", "centered_start"):
        assert calls.get(name, 0) > 0, calls
