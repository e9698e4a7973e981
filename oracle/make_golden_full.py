"""Full-size iterate goldens from the REAL reference (TEST INFRASTRUCTURE).

Runs only in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \
        python oracle/make_golden_full.py config4      # 5M x 10M, 199.9M nnz
    ... python oracle/make_golden_full.py config2      # 500k x 1.15M, 17.9M nnz

The models are the seeded generators of ``paper_2603_03150_b200.instances``
at full scale (config4 seed 4 = the bench instance; config2 seed 2), handed
to ``hybridlp.run_pdhg`` unscaled exactly as the GPU test hands them to the
engine (the GPU box regenerates them from the seed; nothing of the reference
travels).  The full vectors are too large to commit (config 4: 240 MB per
iterate), so per captured iterate the file keeps

  * the 2-norms of x, y, avg_x, avg_y (numpy.linalg.norm, i.e. OpenBLAS);
  * 4,096 entries of each at fixed seeded positions (``sample_idx``);

for k in {1, 2, 64, 65, 100}, plus ``estimate_opnorm(A, seed=0)``
(pdhg.py:80-109, the reference's own power iteration -- the GPU test must
reproduce it without an override), and the state right after the
iteration-64 check (pdhg.py:198-247): restarts, omega, avg_weight and the
restart score, captured as the pre-step state of iteration 65.

Per-iterate capture wraps ``hybridlp.pdhg.pdhg_step``, which ``run_pdhg``
resolves from module globals (pdhg.py:192).  The check scores at iteration
64 are captured by wrapping ``hybridlp.pdhg._score`` (pdhg.py:154-159).
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np
import scipy

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import hybridlp  # noqa: E402
from hybridlp import pdhg as ref_pdhg  # noqa: E402

KEEP = (1, 2, 64, 65, 100)
N_SAMPLE = 4096


def sample_idx(size: int, seed: int) -> np.ndarray:
    return np.sort(np.random.default_rng(seed).choice(size, N_SAMPLE, replace=False))


def main(which: str):
    from paper_2603_03150_b200 import instances

    t0 = time.perf_counter()
    if which == "config4":
        inst = instances.config4(1.0, seed=4)
    elif which == "config2":
        inst = instances.config2(1.0, seed=2)
    else:
        raise SystemExit(f"unknown config {which}")
    p = hybridlp.StandardLp(inst.A, inst.b, inst.c)
    t_gen = time.perf_counter() - t0
    ix, iy = sample_idx(p.n, 100), sample_idx(p.m, 101)
    out = {"m": np.int64(p.m), "n": np.int64(p.n), "nnz": np.int64(p.A.nnz),
           "sample_x": ix, "sample_y": iy,
           "numpy": np.__version__, "scipy": scipy.__version__}

    t = time.perf_counter()
    out["opnorm"] = np.float64(ref_pdhg.estimate_opnorm(p.A, seed=0))
    t_opnorm = time.perf_counter() - t
    print(f"{which}: gen {t_gen:.1f}s opnorm {out['opnorm']!r} in {t_opnorm:.1f}s", flush=True)

    orig_step, orig_score = ref_pdhg.pdhg_step, ref_pdhg._score
    scores = []

    def rec(tag, st):
        for name in ("x", "y", "avg_x", "avg_y"):
            v = getattr(st, name)
            out[f"{tag}_{name}_norm"] = np.float64(np.linalg.norm(v))
            out[f"{tag}_{name}_s"] = v[ix if name.endswith("x") else iy].copy()
        out[f"{tag}_omega"] = np.float64(st.omega)
        out[f"{tag}_restarts"] = np.int64(st.restarts)
        out[f"{tag}_avg_weight"] = np.float64(st.avg_weight)
        out[f"{tag}_restart_score"] = np.float64(st.restart_score)

    def step(state, model):
        if state.iterations == 64:          # state after the iteration-64 check
            rec("post64", state)
        r = orig_step(state, model)
        if state.iterations in KEEP:
            rec(f"k{state.iterations}", state)
            print(f"  k={state.iterations} {time.perf_counter() - t0:.0f}s", flush=True)
        return r

    def score(pp, x, y):
        r = orig_score(pp, x, y)
        scores.append(r[2].max_violation)
        return r

    ref_pdhg.pdhg_step, ref_pdhg._score = step, score
    try:
        pt, st = hybridlp.run_pdhg(p, hybridlp.PdhgParams(eps_rel=1e-12, max_kkt_passes=100))
    finally:
        ref_pdhg.pdhg_step, ref_pdhg._score = orig_step, orig_score
    # scores: [zero point, cur@64, avg@64]
    out["score_zero"] = np.float64(scores[0])
    out["score64_cur"], out["score64_avg"] = np.float64(scores[1]), np.float64(scores[2])
    out["final_iterations"] = np.int64(st.iterations)
    out["final_restarts"] = np.int64(st.restarts)
    out["seconds"] = np.float64(time.perf_counter() - t0)
    path = ROOT / "tests" / "golden" / f"full_{which}.npz"
    np.savez_compressed(path, **out)
    print(json.dumps({"file": str(path), "opnorm": float(out["opnorm"]),
                      "restarts_post64": int(out["post64_restarts"]),
                      "omega_post64": float(out["post64_omega"]),
                      "scores": [float(s) for s in scores], "seconds": float(out["seconds"])}),
          flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
