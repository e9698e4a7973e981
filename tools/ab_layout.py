"""Interleaved A/B timing of step layouts on config 4 (dev tool).

    python tools/ab_layout.py [--variants natural,rows,rows_csr] [--rounds 6]

Builds every variant's device layout once, then alternates: each round times
3 periods (64 iterations, graph) of every variant in turn, so clock and power
drift hit all variants alike; prints the per-variant median ms/iteration and
the SM clock seen during the run.
"""
from __future__ import annotations

import argparse
import json
import statistics
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

VARIANTS = {
    "natural": dict(row_order="natural"),
    "rows": dict(row_order="length"),
    "rows_plain": dict(row_order="length", row_order_first=0),
    "rows_nocol": dict(row_order="length", col_order="natural"),
    "rows_col0": dict(row_order="length", col_order_first=0),
    "rows_colclasses": dict(row_order="length", col_order_first=-1),
    "rows_w16k": dict(row_order="length", row_order_window=16384),
    "rows_w4k": dict(row_order="length", row_order_window=4096),
    "rows_w8k": dict(row_order="length", row_order_window=8192),
    "rows_w32k": dict(row_order="length", row_order_window=32768),
    "rows_w256k": dict(row_order="length", row_order_window=262144),
    "rows_col16": dict(row_order="length", col_order_first=16),
    "rows_col32": dict(row_order="length", col_order_first=32),
    "rows_first64": dict(row_order="length", row_order_first=64),
    "rows_first16": dict(row_order="length", row_order_first=16),
    "rows_first32": dict(row_order="length", row_order_first=32),
    "rows_classes": dict(row_order="length", row_order_first=-1),
    "rows_first48": dict(row_order="length", row_order_first=48),
    "rows_first24": dict(row_order="length", row_order_first=24),
    # experiment build only (PDHG_B200_LIB=tools/_libs/libpdhg_b200_exp.so): L2 persisting windows
    "rows_l2x": dict(row_order="length", l2_persist=2),
    "rows_l2y": dict(row_order="length", l2_persist=1),
    "rows_l2xy": dict(row_order="length", l2_persist=3),
    "rows_csr": dict(row_order="length", sell="off"),
    "csr": dict(row_order="natural", sell="off"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="natural,rows,rows_csr")
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--scale", type=float, default=1.0)
    args = ap.parse_args()
    import torch

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.engine import _start_vector
    from paper_2603_03150_b200.instances import config4

    inst = config4(scale=args.scale, seed=4)
    names = args.variants.split(",")
    devs = {}
    for nm in names:
        d = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False, **VARIANTS[nm]))
        lam = d.opnorm(_start_vector(d.n, 0))
        d.reset()
        devs[nm] = (d, 1.0 / (1.05 * lam))
        d.run_period(64, 0, devs[nm][1], devs[nm][1], 0.0)   # capture the graph
    torch.cuda.synchronize()
    res = {nm: [] for nm in names}
    res_chk = {nm: [] for nm in names}
    from paper_2603_03150_b200 import _native as N
    clocks = []
    for r in range(args.rounds):
        # rotate the order every round: the variant timed first after the previous
        # round sees a different power/clock transition than the others
        order = names[r % len(names):] + names[:r % len(names)]
        for nm in order:
            d, st = devs[nm]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(d.stream)
            for k in range(3):
                d.run_period(64, 64 * (k + 1), st, st, float(64 * (k + 1)))
            e1.record(d.stream)
            torch.cuda.synchronize()
            res[nm].append(e0.elapsed_time(e1) / (3 * 64))
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(d.stream)
            d.check(N.PT_CUR, N.PT_AVG)
            c1.record(d.stream)
            torch.cuda.synchronize()
            res_chk[nm].append(c0.elapsed_time(c1))
        q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                           capture_output=True, text=True).stdout.strip()
        clocks.append(q)
    out = {nm: {"ms_per_iter_median": statistics.median(v), "check_ms_median": statistics.median(res_chk[nm]),
                "all": v} for nm, v in res.items()}
    out["clocks"] = clocks
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
