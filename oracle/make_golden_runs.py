"""Full-size reference runs for BASELINE configs (TEST INFRASTRUCTURE).

Runs the REAL reference (in this container only) through its own pipeline
pieces -- to_standard_form, ruiz_equilibrate, run_pdhg at eps_rel=1e-4 --
on a full-size seeded instance and stores the run summary (status,
iterations, restarts, objective, termination sides, wall time) as JSON
under tests/golden/, so the GPU tests can compare iteration counts and
objectives at full size without the reference:

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 python oracle/make_golden_runs.py config1
    ... python oracle/make_golden_runs.py config4 1.0 nolimit

The third argument ``nolimit`` passes ``time_limit_s=1e9`` (the reference's
default of 10,000 s, pdhg.py:36, stops config 2 at ~48k and config 4 at ~3.5k
iterations on one core) and writes ``run_<config>_s<scale>_nolimit.json``;
``tl=SECONDS`` passes that limit and writes ``run_<config>_s<scale>_tl<SECONDS>.json``
(config 4 needs ~2.8 s per iteration on one core: ~10 h to 1e-4).
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import hybridlp  # noqa: E402

from paper_2603_03150_b200.instances import config1_general, config3_general  # noqa: E402


def main(which: str, scale: float = 1.0, limit: str = ""):
    t0 = time.perf_counter()
    if which in ("config2", "config4"):   # built directly in standard form
        from paper_2603_03150_b200 import instances

        inst = getattr(instances, which)(scale)
        p = hybridlp.StandardLp(inst.A, inst.b, inst.c)
        del inst
    else:
        g = (config1_general if which == "config1" else config3_general)(scale).to_reference()
        t0 = time.perf_counter()
        p, fmap = hybridlp.to_standard_form(g)
    t1 = time.perf_counter()
    s, info = hybridlp.ruiz_equilibrate(p)
    t2 = time.perf_counter()
    orig_score, n_scores = hybridlp.pdhg._score, [0]

    def score(pp, x, y):     # progress line every 16 checks (pdhg.py:154-159 unchanged)
        n_scores[0] += 1
        if n_scores[0] % 32 == 0:
            print(f"  {which}: check {n_scores[0] // 2} ({time.perf_counter() - t2:.0f} s)", flush=True)
        return orig_score(pp, x, y)

    hybridlp.pdhg._score = score
    if limit == "nolimit":
        params, suffix = hybridlp.PdhgParams(eps_rel=1e-4, time_limit_s=1e9), "_nolimit"
    elif limit.startswith("tl="):
        tl = float(limit[3:])
        params, suffix = hybridlp.PdhgParams(eps_rel=1e-4, time_limit_s=tl), f"_tl{tl:g}"
    else:
        params, suffix = hybridlp.PdhgParams(eps_rel=1e-4), ""
    pt, st = hybridlp.run_pdhg(s, params)
    t3 = time.perf_counter()
    term = st.termination
    out = {
        "instance": f"{which}{'' if which in ('config2', 'config4') else '_general'}(scale={scale})", "m_std": p.m, "n_std": p.n, "nnz_std": int(p.A.nnz),
        "status": st.status.value, "iterations": st.iterations, "restarts": st.restarts,
        "objective_scaled": float(s.c @ pt.x), "max_violation": st.max_violation,
        "termination": [term.primal_lhs, term.primal_rhs, term.dual_lhs, term.dual_rhs,
                        term.gap_lhs, term.gap_rhs],
        "ruiz_passes": info.applied_iterations,
        "seconds": {"to_standard_form": t1 - t0, "ruiz": t2 - t1, "run_pdhg": t3 - t2},
        "numpy": np.__version__, "threads": "OPENBLAS_NUM_THREADS=1",
        "time_limit_s": params.time_limit_s,
    }
    path = ROOT / "tests" / "golden" / f"run_{which}_s{scale:g}{suffix}.json"
    path.write_text(json.dumps(out, indent=1))
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0, sys.argv[3] if len(sys.argv) > 3 else "")
