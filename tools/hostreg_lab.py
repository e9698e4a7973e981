"""Lab: H2D of a 1.6 GB pageable numpy array -- the pinned staging ring
(hostio.h2d) vs page-locking the array in place (cudaHostRegister) and one
DMA, with the registration cost counted."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_03150_b200 import hostio  # noqa: E402

dev = torch.device("cuda", 0)
a = np.random.default_rng(0).standard_normal(200_000_000)
cudart = torch.cuda.cudart()
out = torch.empty(a.size, dtype=torch.float64, device=dev)
torch.cuda.synchronize()
for r in range(3):
    t = time.perf_counter()
    hostio.h2d(a, np.float64, dev)
    torch.cuda.synchronize()
    t_ring = time.perf_counter() - t
    t = time.perf_counter()
    rc = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t_reg = time.perf_counter() - t
    t = time.perf_counter()
    out.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    t_dma = time.perf_counter() - t
    t = time.perf_counter()
    cudart.cudaHostUnregister(a.ctypes.data)
    t_unreg = time.perf_counter() - t
    print({"ring_s": round(t_ring, 4), "ring_GBs": round(a.nbytes / t_ring / 1e9, 1), "register_s": round(t_reg, 4),
           "rc": int(rc), "dma_s": round(t_dma, 4), "dma_GBs": round(a.nbytes / t_dma / 1e9, 1),
           "unregister_s": round(t_unreg, 4),
           "registered_total_GBs": round(a.nbytes / (t_reg + t_dma + t_unreg) / 1e9, 1)}, flush=True)
