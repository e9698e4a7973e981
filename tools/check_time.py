"""Two-point KKT check time on config 4 (and its scalars, for A/B parity).
    python tools/check_time.py [--lib path]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, ".")
if "--lib" in sys.argv:
    from paper_2603_03150_b200 import _native

    _native.LIB_PATH = Path(sys.argv[sys.argv.index("--lib") + 1]).resolve()
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_03150_b200 as eng  # noqa: E402
from paper_2603_03150_b200 import _native as N  # noqa: E402
from paper_2603_03150_b200.engine import _start_vector  # noqa: E402
from paper_2603_03150_b200.instances import config4  # noqa: E402

inst = config4(1.0)
dev = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False))
lam = dev.opnorm(_start_vector(dev.n, 0))
st = 1.0 / (1.05 * lam)
dev.reset()
for r in range(3):
    dev.run_period(64, 64 * r, st, st, float(64 * r))
q = dev.check(N.PT_CUR, N.PT_AVG)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    t = time.perf_counter()
    dev.check(N.PT_CUR, N.PT_AVG)
    ts.append(time.perf_counter() - t)
print(f"lib={N.LIB_PATH.name} check 2pt: min {1e3 * min(ts):.3f} ms median {1e3 * sorted(ts)[5]:.3f} ms")
print("scalars", np.asarray(q).ravel().tolist())
