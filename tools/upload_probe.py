"""How fast can a 2.4 GB CSR reach the device? (dev tool)"""
import time
import numpy as np
import torch

n = 200_000_000
val = np.random.default_rng(0).standard_normal(n)
col = np.arange(n, dtype=np.int32)
dev = torch.device("cuda", 0)
torch.cuda.synchronize()
for rep in range(2):
    t = time.perf_counter()
    a = torch.from_numpy(val).to(dev)
    b = torch.from_numpy(col).to(dev)
    torch.cuda.synchronize()
    print(f"plain .to: {time.perf_counter() - t:.3f} s")
    del a, b
cr = torch.cuda.cudart()
for rep in range(2):
    t = time.perf_counter()
    for arr in (val, col):
        rc = cr.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
        assert int(rc) == 0, rc
    t1 = time.perf_counter()
    ta, tb = torch.from_numpy(val), torch.from_numpy(col)
    print("pinned?", ta.is_pinned())
    a = torch.empty(n, dtype=torch.float64, device=dev)
    b = torch.empty(n, dtype=torch.int32, device=dev)
    a.copy_(ta, non_blocking=True)
    b.copy_(tb, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for arr in (val, col):
        cr.cudaHostUnregister(arr.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {t1 - t:.3f} s, copy {t2 - t1:.3f} s, unregister {t3 - t2:.3f} s, total {t3 - t:.3f}")
    del a, b
