"""Step-kernel times (primal, dual, one iteration) on several BASELINE instances (dev tool).

    python tools/kernel_times.py [--lib path/to/libpdhg_b200.so] [--opts JSON]
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--opts", default="{}")
    ap.add_argument("--full4", action="store_true")
    args = ap.parse_args()
    if args.lib:
        from paper_2603_03150_b200 import _native

        _native.LIB_PATH = Path(args.lib).resolve()
    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.instances import config1_general, config2, config3_general, config4

    kw = json.loads(args.opts)
    models = {}
    p, _ = eng.to_standard_form(config1_general(1.0))
    models["config1"] = eng.ruiz_equilibrate(p, register_layout=False)[0]
    models["config2"] = eng.ruiz_equilibrate(config2(1.0), register_layout=False)[0]
    p, _ = eng.to_standard_form(config3_general(1.0))
    models["config3"] = p
    models["config4_s0.05"] = config4(0.05)
    if "--full4" in sys.argv:
        models["config4"] = config4(1.0)
    for name, m in models.items():
        dev = eng.DeviceLp(m.A, m.b, m.c, eng.GpuOptions(cache_layout=False, **kw))
        dev.reset()
        row = {"model": name, "nnz": int(m.A.nnz), "lanes": [dev.a_lanes, dev.at_lanes],
               "sell": {k: v["used"] for k, v in dev.sell_info.items()},
               "primal_us": 1e3 * dev.time_kernel(0, 50, 1e-3, 1e-3),
               "dual_us": 1e3 * dev.time_kernel(1, 50, 1e-3, 1e-3),
               "iter_us": 1e3 * dev.time_kernel(2, 50, 1e-3, 1e-3)}
        import time

        import torch

        from paper_2603_03150_b200 import _native as N

        dev.check(N.PT_CUR, N.PT_AVG)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(10):
            dev.check(N.PT_CUR, N.PT_AVG)
        row["check_us"] = 1e6 * (time.perf_counter() - t) / 10
        print(json.dumps(row), flush=True)
        del dev


if __name__ == "__main__":
    main()
