import sys, time, json
sys.path.insert(0, ".")
import torch
import paper_2603_03150_b200 as eng
from paper_2603_03150_b200.instances import config4
inst = config4(1.0)
for k in range(3):
    t = time.perf_counter()
    d = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False))
    torch.cuda.synchronize()
    print(k, round(time.perf_counter() - t, 3), json.dumps(d.timings), flush=True)
    del d
for k in range(2):
    t = time.perf_counter()
    d = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False, row_order="natural"))
    torch.cuda.synchronize()
    print("natural", k, round(time.perf_counter() - t, 3), json.dumps(d.timings), flush=True)
    del d
