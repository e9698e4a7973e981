"""Generate tests/golden/*.npz from the REAL reference (TEST INFRASTRUCTURE).

Runs only in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py

It imports ``hybridlp`` from /root/reference/pkg/src and the desk-instance
builders from /root/reference/pkg/tests/_desk.py, builds the standard-form
models the reference hands to run_pdhg, and records, per instance:

  * the model itself (A as CSR arrays, b, c) -- so the GPU box needs no reference;
  * estimate_opnorm(A, seed=0) and one A@v / A'w pair (the 1e-12 SpMV gate);
  * the first 100 PDHG iterates of run_pdhg (x, y, avg_x, avg_y, omega,
    restarts), captured by wrapping hybridlp.pdhg.pdhg_step, which run_pdhg
    resolves from module globals (pdhg.py:192);
  * full-run results (status, iterations, restarts, termination sides,
    max_violation, objective, final x/y/z) at several tolerances, plus
    IterationLimit runs (max_kkt_passes=128) that exercise the best-point
    return path (pdhg.py:249-258).

numpy/scipy versions are stored with every file.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import scipy

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"

sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))
sys.path.insert(0, str(ROOT))

import hybridlp  # noqa: E402
from hybridlp import pdhg as ref_pdhg  # noqa: E402
from _desk import lp1, lp2, planted_equality_lp, planted_inequality_lp  # noqa: E402

from paper_2603_03150_b200.instances import config0_general  # noqa: E402

CAPTURE = 100


def models():
    out = {}
    p, _ = hybridlp.to_standard_form(lp1().model)
    out["lp1_std"] = p
    p, _ = hybridlp.to_standard_form(lp2().model)
    out["lp2_ruiz"], _ = hybridlp.ruiz_equilibrate(p)
    for m, n, s in ((10, 18, 7), (20, 35, 17), (40, 70, 20)):
        p, _ = hybridlp.to_standard_form(planted_equality_lp(m, n, s).model)
        out[f"eq_{m}x{n}_s{s}_ruiz"], _ = hybridlp.ruiz_equilibrate(p)
    p, _ = hybridlp.to_standard_form(planted_inequality_lp(12, 20, 32).model)
    out["ineq_12x20_s32_ruiz"], _ = hybridlp.ruiz_equilibrate(p)
    # BASELINE config 0 through the reference pipeline's own preparation
    A, b, c, _, _ = config0_general(seed=0)
    g = hybridlp.GeneralLp(c=c, A=A, senses=[hybridlp.EQ] * A.shape[0], rhs=b,
                           lower=np.zeros(A.shape[1]), upper=np.full(A.shape[1], np.inf))
    prep = hybridlp.warmstart.prepare_model(g)
    out["config0_s0"] = prep.solve_model
    return out


def capture_iterates(p, params, seed=0, keep=None):
    rec = []
    orig = ref_pdhg.pdhg_step

    def wrapped(state, model):
        r = orig(state, model)
        if state.iterations <= CAPTURE and (keep is None or state.iterations in keep):
            rec.append((state.iterations, state.x.copy(), state.y.copy(), state.avg_x.copy(),
                        state.avg_y.copy(), state.omega, state.restarts, state.avg_weight))
        return r

    ref_pdhg.pdhg_step = wrapped
    try:
        hybridlp.run_pdhg(p, params, seed=seed)
    finally:
        ref_pdhg.pdhg_step = orig
    return rec


def run_record(p, params, seed=0):
    pt, st = hybridlp.run_pdhg(p, params, seed=seed)
    t = st.termination
    return {
        "status": st.status.value, "iterations": st.iterations, "restarts": st.restarts,
        "max_violation": st.max_violation,
        "term": np.array([t.primal_lhs, t.primal_rhs, t.dual_lhs, t.dual_rhs, t.gap_lhs, t.gap_rhs]),
        "term_ok": bool(t.ok), "obj": float(p.c @ pt.x), "x": pt.x, "y": pt.y, "z": pt.z,
    }


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(123)
    for name, p in models().items():
        A = p.A.tocsr()
        d = {
            "numpy_version": np.__version__, "scipy_version": scipy.__version__,
            "A_data": A.data, "A_indices": A.indices, "A_indptr": A.indptr,
            "A_shape": np.array(A.shape), "b": p.b, "c": p.c,
            "opnorm_seed0": hybridlp.estimate_opnorm(A, seed=0),
        }
        v = rng.standard_normal(p.n)
        w = rng.standard_normal(p.m)
        d["spmv_v"], d["spmv_Av"] = v, A @ v
        d["spmv_w"], d["spmv_Atw"] = w, p.at_y(w)
        keep = None
        if p.n > 300:
            keep = {1, 2, 3, 4, 8, 16, 32, 63, 64, 65, 66, 96, 100}
        it = capture_iterates(p, hybridlp.PdhgParams(eps_rel=1e-12, max_kkt_passes=CAPTURE), keep=keep)
        d["it_k"] = np.array([r[0] for r in it])
        for j, key in enumerate(("it_x", "it_y", "it_avgx", "it_avgy"), start=1):
            d[key] = np.stack([r[j] for r in it])
        d["it_omega"] = np.array([r[5] for r in it])
        d["it_restarts"] = np.array([r[6] for r in it])
        d["it_avgw"] = np.array([r[7] for r in it])
        runs = [("e4", hybridlp.PdhgParams(eps_rel=1e-4)),
                ("e6", hybridlp.PdhgParams(eps_rel=1e-6)),
                ("lim128", hybridlp.PdhgParams(eps_rel=1e-12, max_kkt_passes=128)),
                ("lim200", hybridlp.PdhgParams(eps_rel=1e-12, max_kkt_passes=200))]
        if p.n <= 300:
            runs.append(("e8", hybridlp.PdhgParams(eps_rel=1e-8)))
        for tag, prm in runs:
            r = run_record(p, prm)
            for k, val in r.items():
                d[f"run_{tag}_{k}"] = np.asarray(val)
        np.savez_compressed(OUT / f"{name}.npz", **d)
        print(f"{name}: m={p.m} n={p.n} nnz={A.nnz} e4 iters={int(d['run_e4_iterations'])} "
              f"restarts={int(d['run_e4_restarts'])} status={d['run_e4_status']}")


if __name__ == "__main__" and "--ruiz" not in sys.argv:
    main()


def ruiz_models():
    """Unscaled standard-form models the reference's prepare_model would
    equilibrate (transform.py:35-77), for the GPU Ruiz parity gate."""
    out = {}
    p, _ = hybridlp.to_standard_form(lp2().model)
    out["ruiz_lp2"] = p
    p, _ = hybridlp.to_standard_form(planted_equality_lp(40, 70, 20).model)
    out["ruiz_eq_40x70"] = p
    p, _ = hybridlp.to_standard_form(planted_inequality_lp(35, 60, 34).model)
    out["ruiz_ineq_35x60"] = p
    A, b, c, _, _ = config0_general(seed=0)
    g = hybridlp.GeneralLp(c=c, A=A, senses=[hybridlp.EQ] * A.shape[0], rhs=b,
                           lower=np.zeros(A.shape[1]), upper=np.full(A.shape[1], np.inf))
    prep = hybridlp.warmstart.prepare_model(g, use_scaling=False)
    out["ruiz_config0"] = prep.solve_model
    return out


def main_ruiz():
    for name, p in ruiz_models().items():
        A = p.A.tocsr()
        scaled, info = hybridlp.ruiz_equilibrate(p)
        S = scaled.A.tocsr()
        np.savez_compressed(
            OUT / f"{name}.npz",
            numpy_version=np.__version__, scipy_version=scipy.__version__,
            A_data=A.data, A_indices=A.indices, A_indptr=A.indptr, A_shape=np.array(A.shape),
            b=p.b, c=p.c, row_scale=info.row_scale, col_scale=info.col_scale,
            applied=np.array(info.applied_iterations), S_data=S.data, S_indices=S.indices,
            S_indptr=S.indptr, Sb=scaled.b, Sc=scaled.c)
        print(f"{name}: m={p.m} n={p.n} nnz={A.nnz} applied={info.applied_iterations}")


if __name__ == "__main__" and "--ruiz" in sys.argv:
    main_ruiz()
