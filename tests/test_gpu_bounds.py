"""Memory safety of the hand-written kernels without compute-sanitizer (closed
on the GPU pool): the bounds-checked build of the library
(tools/_libs/libpdhg_b200_checked.so, built by __graft_entry__.build() with
-DPDHG_BOUNDS_CHECK=1) checks every gathered-vector index, matrix-stream
index and sliced-ELL slot against its bound on the device.  The workload
(tools/sanitize_run.py) drives every default step and check kernel, the
layouts the automatic choice can select, the sharded loopback paths (copy,
fused peer stores, overlapped split steps), Ruiz, standard form and the
finishing kernels; it must report zero out-of-bounds loads."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CHECKED = ROOT / "tools" / "_libs" / "libpdhg_b200_checked.so"


def test_bounds_checked_workload_has_no_out_of_bounds_loads():
    if not CHECKED.exists():
        pytest.skip("bounds-checked build missing (python -m paper_2603_03150_b200.build --checked)")
    env = dict(os.environ, PDHG_B200_LIB=str(CHECKED), PYTHONDONTWRITEBYTECODE="1")
    res = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_run.py")], env=env, cwd=str(ROOT),
                         capture_output=True, text=True, timeout=1200)
    out = res.stdout + res.stderr
    log = ROOT / "gpurun_out"
    if log.is_dir():
        (log / "bounds_check.log").write_text(out)
    assert res.returncode == 0, out[-4000:]
    assert "bounds-checked build: True; out-of-bounds loads: 0" in out, out[-4000:]
