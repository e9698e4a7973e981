"""Lab: where a run_pdhg call's setup goes on config 4 (upload, layout steps,
power iteration, download) -- three calls of 64 iterations from host arrays.

    python tools/setup_profile.py [--scale 1.0]
"""
from __future__ import annotations

import argparse

import numpy as np
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    args = ap.parse_args()
    import torch

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.instances import config4

    inst = config4(scale=args.scale, seed=4)
    T = eng.types()
    from paper_2603_03150_b200 import hostio

    for r in range(4):
        torch.cuda.synchronize()
        ms0 = torch.cuda.memory_stats()
        t0 = time.perf_counter()
        pt, st = eng.run_pdhg(inst, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=64),
                              gpu=eng.GpuOptions(cache_layout=False))
        torch.cuda.synchronize()
        ms1 = torch.cuda.memory_stats()
        segs = ms1.get("segment.all.allocated", 0) - ms0.get("segment.all.allocated", 0)
        print(json.dumps({"call": r, "wall_s": round(time.perf_counter() - t0, 4), "new_segments": segs,
                          "reserved_gb": round(ms1.get("reserved_bytes.all.current", 0) / 1e9, 2),
                          "timings": st.timings}), flush=True)
    # the upload alone, array by array
    for r in range(3):
        out = {}
        for name, a, dt in (("indptr", inst.A.indptr, np.int32), ("indices", inst.A.indices, np.int32),
                            ("data", inst.A.data, np.float64)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            t = hostio.h2d(a, dt, torch.device("cuda", 0))
            torch.cuda.synchronize()
            out[name] = round(time.perf_counter() - t0, 4)
            del t
        print(json.dumps({"h2d_round": r, "s": out}), flush=True)


if __name__ == "__main__":
    main()
