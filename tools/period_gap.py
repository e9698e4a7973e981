"""Lab: how much of a period is host round trip?  Config 4, the product's
run_period_check per period (as bench.py and engine._run call it), with CUDA
events recorded before and after every call on the engine stream:

  busy = e_after[k] - e_before[k]   (graph + check + copies, + enqueue latency)
  gap  = e_before[k+1] - e_after[k] (host time between two calls)

and the same periods through engine._run's own decision logic (run_pdhg with
check_every=64 for a fixed number of iterations, wall clock).

    python tools/period_gap.py [--scale 1.0] [--periods 10]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--periods", type=int, default=10)
    args = ap.parse_args()
    import torch

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200 import _native as N
    from paper_2603_03150_b200.engine import _start_vector
    from paper_2603_03150_b200.instances import config4

    inst = config4(scale=args.scale, seed=4)
    d = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False))
    lam = d.opnorm(_start_vector(d.n, 0))
    st = 1.0 / (1.05 * lam)
    d.reset()
    it = 0
    for _ in range(3):
        d.run_period_check(64, it, st, st, float(it), N.PT_CUR, N.PT_AVG)
        it += 64
    s = d.stream
    K = args.periods
    eb = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ea = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    host_call = []
    for k in range(K):
        eb[k].record(s)
        h0 = time.perf_counter()
        d.run_period_check(64, it, st, st, float(it), N.PT_CUR, N.PT_AVG)
        host_call.append(time.perf_counter() - h0)
        ea[k].record(s)
        it += 64
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    busy = [eb[k].elapsed_time(ea[k]) for k in range(K)]
    gap = [ea[k].elapsed_time(eb[k + 1]) for k in range(K - 1)]
    total = eb[0].elapsed_time(ea[-1])
    out = {"periods": K, "total_ms": total, "wall_ms": wall * 1e3,
           "busy_ms_median": statistics.median(busy), "gap_ms_median": statistics.median(gap),
           "gap_ms": gap, "host_call_ms_median": 1e3 * statistics.median(host_call)}
    # graph and check separately (events around each, one period)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(s)
    d.run_period(64, it, st, st, float(it))
    e[1].record(s)
    d.check(N.PT_CUR, N.PT_AVG)
    e[2].record(s)
    torch.cuda.synchronize()
    out["graph_ms"] = e[0].elapsed_time(e[1])
    out["check_ms"] = e[1].elapsed_time(e[2])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
