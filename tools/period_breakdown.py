"""Where a config-4 period goes: isolated step kernels, one alternating
iteration, the 64-iteration graph without / with the 2-point check, and the
same after a sustained (power-capped) stretch.  python tools/period_breakdown.py"""
import subprocess
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2603_03150_b200 as eng  # noqa: E402
from paper_2603_03150_b200 import _native as N  # noqa: E402
from paper_2603_03150_b200.instances import config4  # noqa: E402

inst = config4(1.0)
dev = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False))
from paper_2603_03150_b200.engine import _start_vector  # noqa: E402

lam = dev.opnorm(_start_vector(dev.n, 0))
dev.reset()
tw = sw = 1.0 / (1.05 * lam)      # the run's real step sizes (omega = 1): iterates stay finite


def clocks():
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                       capture_output=True, text=True).stdout.strip()
    return q


def period_ms(check: bool, reps=5):
    st = torch.cuda.current_stream()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for r in range(reps):
        if check:
            dev.run_period_check(64, 64 * r, tw, sw, 0.0, N.PT_CUR, N.PT_AVG)
        else:
            dev.run_period(64, 64 * r, tw, sw, 0.0)
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t) / reps


def report(tag):
    dev.reset()
    p = dev.time_kernel(0, 30, tw, sw)
    d = dev.time_kernel(1, 30, tw, sw)
    it = dev.time_kernel(2, 30, tw, sw)
    pn = period_ms(False)
    pc = period_ms(True)
    print(f"[{tag}] clocks/power {clocks()} | primal {p:.3f} dual {d:.3f} sum {p + d:.3f} | "
          f"alternating iteration {it:.3f} | period graph {pn:.1f} ms = {pn / 64:.3f}/it | "
          f"period+check {pc:.1f} ms = {pc / 64:.3f}/it (check {pc - pn:.2f} ms)", flush=True)


period_ms(True, 2)
report("cold")
# the bench's order: real periods from a reset state, then the kernels alone
dev.reset()
for r in range(13):
    dev.run_period(64, 64 * r, tw, sw, float(64 * r))
    dev.check(N.PT_CUR, N.PT_AVG)
torch.cuda.synchronize()
print(f"[bench order] after 13 periods: primal {dev.time_kernel(0, 20, tw, sw):.3f} dual "
      f"{dev.time_kernel(1, 20, tw, sw):.3f} iteration {dev.time_kernel(2, 20, tw, sw):.3f}", flush=True)
print(f"[bench order] again: primal {dev.time_kernel(0, 20, tw, sw):.3f} dual "
      f"{dev.time_kernel(1, 20, tw, sw):.3f}", flush=True)
dev.reset()
print(f"[after reset] primal {dev.time_kernel(0, 20, tw, sw):.3f} dual "
      f"{dev.time_kernel(1, 20, tw, sw):.3f}", flush=True)
t = time.time()
while time.time() - t < 20:
    dev.run_period_check(64, 0, tw, sw, 0.0, N.PT_CUR, N.PT_AVG)
report("after 20 s")

sys.path.insert(0, ".")
from bench import live_kernel_ms  # noqa: E402

dev.reset()
for r in range(3):
    dev.run_period(64, 64 * r, tw, sw, float(64 * r))
print("[live events] per-kernel", live_kernel_ms(dev, 192, tw), flush=True)
print(f"[graph] period {period_ms(False):.1f} ms", flush=True)
del dev
torch.cuda.empty_cache()
dev = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False, graphs=False))
dev.reset()
period_ms(False, 2)
print(f"[direct launches] period {period_ms(False):.1f} ms", flush=True)
print("[direct] live per-kernel", live_kernel_ms(dev, 192, tw), flush=True)
