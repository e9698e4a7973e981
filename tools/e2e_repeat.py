"""Repeat the bench's e2e leg (run_pdhg on host arrays, fresh allocator) and
print its phase timings; --sync-v0 generates the start vector inline."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2603_03150_b200 as eng  # noqa: E402
from paper_2603_03150_b200 import engine, hostio  # noqa: E402
from paper_2603_03150_b200.instances import config4  # noqa: E402


class _Sync:
    def submit(self, f, *a):
        class F:
            def __init__(s, v):
                s.v = v

            def result(s):
                return s.v
        return F(f(*a))


inst = config4(scale=1.0)
T = eng.types()
for mode in ("overlap", "sync", "overlap", "sync"):
    eng.clear_cache()
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    real = hostio._executor
    if mode == "sync":
        engine.hostio._executor = lambda: _Sync()
    t = time.perf_counter()
    pt, st = eng.run_pdhg(inst, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=640))
    torch.cuda.synchronize()
    w = time.perf_counter() - t
    hostio._executor = real
    tm = st.timings
    print(f"{mode:8s} wall {w:.3f}  " + "  ".join(f"{k}={v:.3f}" for k, v in tm.items() if isinstance(v, float)),
          {k: round(v, 3) for k, v in tm.get("layout_detail", {}).items()}, flush=True)
