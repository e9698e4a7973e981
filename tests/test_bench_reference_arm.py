"""bench.py's reference arm runs on CPU (the reference's own path from
oracle/_ref, or its pinned port) and prints the contract's JSON line."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--scale", "0.002",
                          "--steps", "2", "--warmup", "1"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "iter/s" and line["value"] > 0
    # the unmodified reference (oracle/_ref, built by oracle/make_ref.sh) or its pinned port
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] == 1
    assert line["config"]["workload"].startswith("config4 (m=10000, n=20000")
    assert line["cpu_baseline"]["host"]["nproc"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["higher_is_better"] is True and line["steps"] == 2 and line["warmup"] == 1
