"""A/B of a library variant on whole periods and runs:
config 4 period (64 iterations, graph) and runs to 1e-4 on configs 1 and 3.
    python tools/period_ab.py [--lib path] [--no4]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, ".")
if "--lib" in sys.argv:
    from paper_2603_03150_b200 import _native

    _native.LIB_PATH = Path(sys.argv[sys.argv.index("--lib") + 1]).resolve()
import torch  # noqa: E402

import paper_2603_03150_b200 as eng  # noqa: E402
from paper_2603_03150_b200 import _native as N  # noqa: E402
from paper_2603_03150_b200.engine import _start_vector  # noqa: E402
from paper_2603_03150_b200.instances import config1_general, config3_general, config4  # noqa: E402

T = eng.types()
out = {"lib": N.LIB_PATH.name}
for name, gen in (("config1", config1_general), ("config3", config3_general)):
    p, _ = eng.to_standard_form(gen(1.0))
    s, _ = eng.ruiz_equilibrate(p)
    eng.run_pdhg(s, T.PdhgParams(eps_rel=1e-4, max_kkt_passes=640))     # warm (graphs, allocator)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        pt, st = eng.run_pdhg(s, T.PdhgParams(eps_rel=1e-4))
        best = min(best, st.timings["iterate_s"])
    out[name] = {"iterations": st.iterations, "iterate_s": round(best, 4),
                 "us_per_iter": round(1e6 * best / st.iterations, 2)}
if "--no4" not in sys.argv:
    inst = config4(1.0)
    dev = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False))
    lam = dev.opnorm(_start_vector(dev.n, 0))
    stp = 1.0 / (1.05 * lam)
    dev.reset()
    for r in range(3):
        dev.run_period(64, 64 * r, stp, stp, float(64 * r))
    torch.cuda.synchronize()
    t = time.perf_counter()
    for r in range(3, 13):
        dev.run_period(64, 64 * r, stp, stp, float(64 * r))
    torch.cuda.synchronize()
    out["config4_period_ms"] = round(1e3 * (time.perf_counter() - t) / 10, 2)
print(out, flush=True)
