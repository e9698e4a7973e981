"""Where a sharded period goes (loopback shards on one GPU, overlapped split
schedule): wall time of run_period (graph + fail-word exchange) and of the
two-point check, with and without the whole-row sliced-ELL layout of the
shards (GpuOptions.split_full_sell: the check's and power iteration's
kernels).  Config 4.

    python tools/sharded_breakdown.py [--scale 1.0] [--G 1] [--periods 5]
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
    ap.add_argument("--G", type=int, default=1)
    ap.add_argument("--periods", type=int, default=5)
    args = ap.parse_args()
    import torch

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200 import _native as N
    from paper_2603_03150_b200.engine import _start_vector
    from paper_2603_03150_b200.instances import config4
    from paper_2603_03150_b200.sharded import build_sharded

    inst = config4(scale=args.scale, seed=4)
    for full in (True, False):
        dev = build_sharded(inst, args.G, "loopback", eng.GpuOptions(split_full_sell=full), overlap="on")
        lam = dev.opnorm(_start_vector(inst.A.shape[1], 0))
        st = 1.0 / (1.05 * lam)
        dev.reset()
        it = 0
        for _ in range(2):
            dev.run_period(64, it, st, st, float(it))
            dev.check(N.PT_CUR, N.PT_AVG)
            it += 64
        per, chk = [], []
        for _ in range(args.periods):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev.run_period(64, it, st, st, float(it))
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            dev.check(N.PT_CUR, N.PT_AVG)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            per.append(1e3 * (t1 - t0))
            chk.append(1e3 * (t2 - t1))
            it += 64
        s0 = dev.shards[0]
        print(json.dumps({"split_full_sell": full, "G": args.G, "scale": args.scale,
                          "full_sell": {k: s0._sell[k] is not None for k in ("A", "At")},
                          "parts": {k: s0._sell_part[k] is not None for k in ("A", "At")},
                          "period_ms": statistics.median(per), "check_ms": statistics.median(chk),
                          "period_ms_all": per, "check_ms_all": chk}), flush=True)
        del dev
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
