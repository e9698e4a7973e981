"""Time the two step kernels on config 4 under each layout/L2 option (dev tool).

    python tools/kernel_matrix.py [--scale 1.0] [--reps 20]
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
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--variants", default="csr,csr_l2d,csr_l2p,csr_l2")
    ap.add_argument("--lib", default=None, help="load this build of libpdhg_b200.so (experiment variants)")
    args = ap.parse_args()
    if args.lib:
        from paper_2603_03150_b200 import _native

        _native.LIB_PATH = Path(args.lib).resolve()
    import numpy as np
    import torch

    import paper_2603_03150_b200 as eng
    from bench import algorithmic_bytes
    from paper_2603_03150_b200.instances import config4

    t = time.time()
    inst = config4(scale=args.scale, seed=4)
    print(f"gen {time.time() - t:.1f}s m={inst.m} n={inst.n} nnz={inst.nnz}", flush=True)
    ab = algorithmic_bytes(inst.m, inst.n, inst.nnz)
    variants = {
        "csr": dict(psr="off", sell="off", l2_persist=0),
        "sell": dict(psr="off", sell="on"),
        "sell_unsorted": dict(psr="off", sell="on", sell_sort="off"),
        "auto": dict(),
        "natural": dict(row_order="natural"),
        "rows": dict(row_order="length"),
        "rows_w4k": dict(row_order="length", row_order_window=4096),
        "rows_global": dict(row_order="length", row_order_window=10**9),
        "rows_h1k": dict(row_order="length", heavy_threshold=1024),
        "direct": dict(graphs=False),
        "auto_sorted": dict(sell_sort="on"),
        "auto_unsorted": dict(sell_sort="off"),
        "persist": dict(psr="off", sell="off", persistent="on"),
        "csr_a8": dict(psr="off", sell="off", a_lanes=8),
        "csr_at16": dict(psr="off", sell="off", at_lanes=16),
        "csr_k1": dict(psr="off", dual_split=1),
        "csr_k3": dict(psr="off", dual_split=3),
        "csr_k4": dict(psr="off", dual_split=4),
        "csr_l2d": dict(psr="off", l2_persist=2),
        "csr_l2p": dict(psr="off", l2_persist=1),
        "csr_l2": dict(psr="off", l2_persist=3),
        "psr": dict(psr="on", l2_persist=0),
        "psr_l2d": dict(psr="on", l2_persist=2),
    }
    out = {}
    for name in args.variants.split(","):
        t = time.time()
        dev = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False, **variants[name]))
        torch.cuda.synchronize()
        build = time.time() - t
        dev.reset()
        tp = dev.time_kernel(0, args.reps, 1e-3, 1e-3)
        td = dev.time_kernel(1, args.reps, 1e-3, 1e-3)
        talt = dev.time_kernel(2, args.reps, 1e-3, 1e-3)
        talt192 = dev.time_kernel(2, 192, 1e-3, 1e-3)   # as long as the 3 graph periods below
        # alternating primal/dual as in a real period (graph of 64 iterations)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dev.run_period(64, 0, 1e-3, 1e-3, 0.0)
        ev0.record(dev.stream)
        for k in range(3):
            dev.run_period(64, 64 * (k + 1), 1e-3, 1e-3, float(64 * (k + 1)))
        ev1.record(dev.stream)
        torch.cuda.synchronize()
        per_iter = ev0.elapsed_time(ev1) / (3 * 64)
        out[name] = {"build_s": build, "primal_ms": tp, "dual_ms": td, "iter_ms": per_iter, "alt_ms": talt, "alt192_ms": talt192,
                     "primal_gbs": ab["primal"] / tp / 1e6, "dual_gbs": ab["dual"] / td / 1e6,
                     "psr": dev.psr_info, "sell": dev.sell_info}
        print(name, json.dumps(out[name]), flush=True)
        del dev
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
