"""Graph vs single-block period kernel on config-4-shaped models of growing size (dev tool)."""

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.instances import config4

    T = eng.types()
    for scale in (0.0002, 0.0005, 0.001, 0.002, 0.005):
        p = config4(scale=scale, seed=7)
        row = {"scale": scale, "m": p.m, "n": p.n, "nnz": p.nnz}
        for mode in ("off", "tiny"):
            opts = eng.GpuOptions(persistent=mode, sell="off")
            params = T.PdhgParams(eps_rel=1e-12, max_kkt_passes=1024)
            eng.run_pdhg(p, params, gpu=opts)
            t = time.perf_counter()
            pt, st = eng.run_pdhg(p, params, gpu=opts)
            row[mode] = {"s": time.perf_counter() - t, "it": st.iterations,
                         "us_per_it": 1e6 * st.timings.get("iterate_s", 0) / max(1, st.iterations)}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
