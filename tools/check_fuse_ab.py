"""A/B (interleaved, one process, one layout): config-4 periods (64 iterations
+ two-point check, run_period_check) with and without the check's A side
fused into the last dual step (pdhg_check_fuse_enable toggled on the same
context; the check -> first primal step reuse stays on).

    python tools/check_fuse_ab.py [--scale 1.0] [--rounds 8] [--periods 3]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--rounds", type=int, default=8)
    ap.add_argument("--periods", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200 import _native as N
    from paper_2603_03150_b200.engine import _start_vector
    from paper_2603_03150_b200.instances import config4

    inst = config4(scale=args.scale, seed=4)
    d = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False))
    assert d.check_dot and d.check_fuse
    lam = d.opnorm(_start_vector(d.n, 0))
    st = 1.0 / (1.05 * lam)
    d.reset()
    it = 0
    s = d.stream
    res = {"on": [], "off": []}

    def periods(on: bool, k: int) -> float:
        nonlocal it
        N.check(d.lib.pdhg_check_fuse_enable(d.ctx, 1 if on else 0))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(k):
            d.run_period_check(64, it, st, st, float(it), N.PT_CUR, N.PT_AVG)
            d.use_check_dot(0)
            it += 64
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k

    periods(True, 2)
    periods(False, 2)
    for r in range(args.rounds):
        for mode in (("on", "off") if r % 2 == 0 else ("off", "on")):
            res[mode].append(periods(mode == "on", args.periods))
    out = {"ms_per_period_median": {k: statistics.median(v) for k, v in res.items()},
           "ms_per_period": res}
    out["gain_pct"] = 100 * (1 - out["ms_per_period_median"]["on"] / out["ms_per_period_median"]["off"])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
