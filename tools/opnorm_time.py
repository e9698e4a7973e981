"""Power iteration on config 4 (k_spmv / k_spmv_sell launches) -- for the ncu launch list."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2603_03150_b200 as eng  # noqa: E402
from paper_2603_03150_b200.engine import _start_vector  # noqa: E402
from paper_2603_03150_b200.instances import config4  # noqa: E402

inst = config4(1.0)
dev = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False))
v0 = _start_vector(dev.n, 0)
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    lam = dev.opnorm(v0)
    torch.cuda.synchronize()
    print(f"opnorm {lam:.6f} in {time.perf_counter() - t:.4f} s", flush=True)
