"""Repeat the bench's e2e leg (run_pdhg on host arrays) and print its phase
timings; the first call runs with a cold allocator, later ones warm."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2603_03150_b200 as eng  # noqa: E402
from paper_2603_03150_b200.instances import config4  # noqa: E402

inst = config4(scale=1.0)
T = eng.types()
for rep in range(3):
    eng.clear_cache()
    torch.cuda.synchronize()
    t = time.perf_counter()
    pt, st = eng.run_pdhg(inst, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=640))
    torch.cuda.synchronize()
    w = time.perf_counter() - t
    tm = st.timings
    print(f"rep {rep} wall {w:.3f}  " + "  ".join(f"{k}={v:.3f}" for k, v in tm.items() if isinstance(v, float)),
          {k: round(v, 3) for k, v in tm.get("layout_detail", {}).items()}, flush=True)
