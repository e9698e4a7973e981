"""Phase times of the device Ruiz on config 4 (host checks, upload, passes,
download, assembly, layout hand-over).  python tools/ruiz_timing.py [scale]"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2603_03150_b200 as eng  # noqa: E402
from paper_2603_03150_b200.instances import config4  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
t = time.perf_counter()
inst = config4(scale=scale)
print(f"instance {time.perf_counter() - t:.2f} s, nnz {inst.A.nnz}", flush=True)
for rep in range(2):
    eng.clear_cache()
    torch.cuda.synchronize()
    t = time.perf_counter()
    scaled, info = eng.ruiz_equilibrate(inst)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t
    print(f"rep {rep}: total {tot:.3f} s passes={info.applied_iterations}",
          {k: round(v, 4) for k, v in eng.ruiz.last_timings.items()}, flush=True)
