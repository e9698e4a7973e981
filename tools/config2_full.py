"""BASELINE config 2 at full size (500k x 1M + slacks, ~18M nnz): device Ruiz +
run_pdhg to 1e-4 on the GPU, and the oracle's per-iteration time on the CPU
(a few pdhg_step calls + one scored check) for the extrapolated reference."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_03150_b200 as eng  # noqa: E402
from paper_2603_03150_b200.instances import config2  # noqa: E402

T = eng.types()
t = time.perf_counter()
inst = config2(1.0)
out = {"m": inst.A.shape[0], "n": inst.A.shape[1], "nnz": int(inst.A.nnz), "gen_s": time.perf_counter() - t}
torch.cuda.synchronize()
t = time.perf_counter()
scaled, info = eng.ruiz_equilibrate(inst)
torch.cuda.synchronize()
out["ruiz_s"] = time.perf_counter() - t
pt, st = eng.run_pdhg(scaled, T.PdhgParams(eps_rel=1e-4, time_limit_s=600.0))
out.update(status=st.status.value, iterations=st.iterations, restarts=st.restarts,
           pdhg_wall_s=st.wall_seconds, obj=float(np.dot(scaled.c, pt.x)))
print(json.dumps(out), flush=True)
if "--cpu" in sys.argv:
    import bench

    cs = bench.cpu_sample(scaled, steps=3)
    out["cpu_per_iter_s"] = cs["per_iter_s"]
    out["cpu_extrapolated_s"] = cs["per_iter_s"] * st.iterations
    print(json.dumps(out), flush=True)
