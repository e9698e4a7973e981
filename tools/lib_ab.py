"""Time one build of libpdhg_b200 (PDHG_B200_LIB) on config 4: isolated step
kernels and the graph of a period (dev tool; run builds back to back).

    PDHG_B200_LIB=tools/_libs/libX.so python tools/lib_ab.py [--scale 1.0]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    args = ap.parse_args()
    import torch

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.engine import _start_vector
    from paper_2603_03150_b200.instances import config4

    inst = config4(scale=args.scale, seed=4)
    d = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False))
    lam = d.opnorm(_start_vector(d.n, 0))
    st = 1.0 / (1.05 * lam)
    d.reset()
    d.run_period(64, 0, st, st, 0.0)
    its = []
    for r in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(d.stream)
        for k in range(3):
            d.run_period(64, 64 * (k + 1), st, st, float(64 * (k + 1)))
        e1.record(d.stream)
        torch.cuda.synchronize()
        its.append(e0.elapsed_time(e1) / 192)
    out = {"lib": Path(os.environ.get("PDHG_B200_LIB", "product")).name,
           "primal_ms": d.time_kernel(0, 20, st, st), "dual_ms": d.time_kernel(1, 20, st, st),
           "iter_ms_median": statistics.median(its), "iter_ms": its,
           "clock": subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                                   capture_output=True, text=True).stdout.strip()}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
