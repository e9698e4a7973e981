"""Device pipeline on a general-form BASELINE config (dev tool):
standard form (csrc/stdform.cu) -> Ruiz (csrc/ruiz.cu) -> run_pdhg -> finishing
(csrc/finish.cu), each step timed; JSON line on stdout.

    python tools/pipeline_run.py config3 [--scale 1.0] [--eps 1e-4] [--limit 600]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["config1", "config3"])
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--eps", type=float, default=1e-4)
    ap.add_argument("--limit", type=float, default=600.0)
    ap.add_argument("--heavy", type=int, default=None, help="GpuOptions.heavy_threshold")
    ap.add_argument("--opts", default="{}", help="GpuOptions fields as JSON")
    args = ap.parse_args()
    import torch

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200 import finish
    from paper_2603_03150_b200.instances import config1_general, config3_general

    T = eng.types()
    f = config1_general if args.which == "config1" else config3_general
    g = f(args.scale) if args.seed is None else f(args.scale, seed=args.seed)
    torch.cuda.synchronize()
    t = {}
    t0 = time.perf_counter()
    p, fmap = eng.to_standard_form(g)
    t["std_form_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    scaled, info = eng.ruiz_equilibrate(p)
    t["ruiz_s"] = time.perf_counter() - t0
    kw = json.loads(args.opts)
    if args.heavy is not None:
        kw["heavy_threshold"] = args.heavy
    opts = eng.GpuOptions(**kw)
    pt, st = eng.run_pdhg(scaled, T.PdhgParams(eps_rel=args.eps, time_limit_s=args.limit), gpu=opts)
    dev = eng.device_lp(scaled, opts)
    t["kernel_ms"] = {"primal": dev.time_kernel(0, 20, 1e-3, 1e-3), "dual": dev.time_kernel(1, 20, 1e-3, 1e-3)}
    t["timings"] = getattr(st, "timings", None)
    t["pdhg_s"] = st.wall_seconds
    t0 = time.perf_counter()
    un = finish.unscale_point(info, pt)
    x, y, z = finish.restrict_point(g, fmap, un)
    viol = finish.evaluate_general_point(g, x, y)
    t["finish_s"] = time.perf_counter() - t0
    out = {"instance": f"{args.which}_general(scale={args.scale})", "opts": kw, "m_std": p.m, "n_std": p.n,
           "nnz_std": int(p.A.nnz), "status": st.status.value, "iterations": st.iterations,
           "restarts": st.restarts, "objective_scaled": float(scaled.c @ pt.x),
           "objective_general": float(g.c @ x), "ruiz_passes": info.applied_iterations,
           "general_violation": {"primal_inf": viol.primal_inf, "dual_inf": viol.dual_inf,
                                 "rel_gap": viol.rel_gap, "max": viol.max_violation},
           "seconds": t, "iters_per_s": st.iterations / max(st.wall_seconds, 1e-9)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
