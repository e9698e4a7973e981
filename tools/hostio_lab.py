"""Host->device / device->host strategies for the model arrays (pageable numpy)."""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_03150_b200 import hostio  # noqa: E402

print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), flush=True)
dev = torch.device("cuda", 0)
a = np.random.default_rng(0).standard_normal(200_000_000)  # 1.6 GB
torch.cuda.synchronize()


def tm(name, f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"{name:40s} {best*1e3:8.1f} ms  {a.nbytes/best/1e9:6.1f} GB/s", flush=True)


tm("torch .to(dev) pageable", lambda: torch.from_numpy(a).to(dev))
tm("hostio.h2d", lambda: hostio.h2d(a, np.float64, dev))
for chunk, nbuf, thr in ((64 << 20, 4, 8), (16 << 20, 8, 8), (32 << 20, 4, 16), (8 << 20, 8, 4)):
    hostio.CHUNK, hostio.NBUF = chunk, nbuf
    hostio._threads = (lambda t=thr: t)
    hostio._pool = None
    hostio._rings.clear()
    tm(f"hostio.h2d chunk={chunk>>20}M nbuf={nbuf} thr={thr}", lambda: hostio.h2d(a, np.float64, dev))
hostio.CHUNK, hostio.NBUF = 32 << 20, 4
hostio._threads = lambda: 8
hostio._pool = None
hostio._rings.clear()
cr = torch.cuda.cudart()


def reg():
    t = torch.from_numpy(a)
    cr.cudaHostRegister(t.data_ptr(), a.nbytes, 0)
    d = t.to(dev, non_blocking=True)
    torch.cuda.synchronize()
    cr.cudaHostUnregister(t.data_ptr())
    return d


tm("cudaHostRegister + copy + unregister", reg)
d = torch.from_numpy(a).to(dev)
tm("d2h torch .cpu()", lambda: d.cpu().numpy())
tm("d2h hostio", lambda: hostio.d2h(d))


def np_copy(thr):
    dst = np.empty_like(a)
    hostio._threads = lambda: thr
    hostio._pool = None
    hostio._par_copy(dst.view(np.uint8), a.view(np.uint8))


for thr in (1, 4, 8, 16):
    tm(f"host par_copy fresh dst thr={thr}", lambda: np_copy(thr))
pin = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
tm("pinned -> device", lambda: pin.to(dev, non_blocking=True))
