"""Run to 1e-4 with the step layouts chosen automatically vs CSR-only on configs 2 and 4 (dev tool)."""

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.instances import config2, config4

    T = eng.types()
    for name, inst in (("config2_s0.1", config2(0.1)), ("config2_s1", config2(1.0)), ("config4_s0.05", config4(0.05))):
        scaled, _ = eng.ruiz_equilibrate(inst)
        for kw in ({"sell": "off"}, {}):
            opts = eng.GpuOptions(cache_layout=False, **kw)
            t = time.perf_counter()
            pt, st = eng.run_pdhg(scaled, T.PdhgParams(eps_rel=1e-4, time_limit_s=600), gpu=opts)
            dev = eng.DeviceLp(scaled.A, scaled.b, scaled.c, opts)
            print(json.dumps({"model": name, "opts": kw, "status": st.status.value, "iterations": st.iterations,
                              "restarts": st.restarts, "pdhg_s": st.wall_seconds, "sell": dev.sell_info,
                              "primal_ms": dev.time_kernel(0, 10, 1e-3, 1e-3),
                              "dual_ms": dev.time_kernel(1, 10, 1e-3, 1e-3)}), flush=True)


if __name__ == "__main__":
    main()
