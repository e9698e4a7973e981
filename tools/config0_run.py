"""Time run_pdhg to 1e-4 on BASELINE config 0 (golden fixture) for GpuOptions variants (dev tool)."""

import json
import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import paper_2603_03150_b200 as eng

    g = np.load(ROOT / "tests" / "golden" / "config0_s0.npz")
    A = sp.csr_matrix((g["A_data"], g["A_indices"], g["A_indptr"]), shape=tuple(g["A_shape"]))

    class P:
        pass

    T = eng.types()
    for kw in ({"sell": "off", "persistent": "off"}, {"sell": "off", "persistent": "on"},
               {"persistent": "tiny"}, {}):
        p = P()
        p.A, p.b, p.c = A, g["b"].copy(), g["c"].copy()
        opts = eng.GpuOptions(**kw)
        eng.run_pdhg(p, T.PdhgParams(eps_rel=1e-4), gpu=opts)   # warm (layout, graphs)
        t = time.perf_counter()
        pt, st = eng.run_pdhg(p, T.PdhgParams(eps_rel=1e-4), gpu=opts)
        dt = time.perf_counter() - t
        print(json.dumps({"opts": kw, "status": st.status.value, "iterations": st.iterations,
                          "restarts": st.restarts, "seconds": dt, "iters_per_s": st.iterations / dt,
                          "timings": st.timings}))


if __name__ == "__main__":
    main()
