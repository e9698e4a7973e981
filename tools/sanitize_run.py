"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): every
default step and check kernel plus the layout variants the auto choice can
select, the sharded loopback paths (copy, fused peer stores, overlapped split
steps), Ruiz, standard form and the finishing kernels -- on small models.

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py
"""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import paper_2603_03150_b200 as eng  # noqa: E402
from conftest import load_golden  # noqa: E402
from paper_2603_03150_b200.instances import config2, config4  # noqa: E402
from paper_2603_03150_b200.sharded import run_pdhg_sharded  # noqa: E402

from paper_2603_03150_b200 import _native as N  # noqa: E402

T = eng.types()
done = []
CHECKED = N.bounds_checked()     # PDHG_B200_LIB=tools/_libs/libpdhg_b200_checked.so
oob_total = 0


def oob(tag):
    """Out-of-bounds loads the checked build saw since the last call."""
    global oob_total
    if not CHECKED:
        return None
    n, i, b = N.debug_oob()
    oob_total += n
    if n:
        print(f"OUT OF BOUNDS after {tag}: {n} loads, first index {i} >= bound {b}", flush=True)
    return n


def run(tag, p, opts=None, **kw):
    pt, st = eng.run_pdhg(p, T.PdhgParams(**kw), gpu=opts or eng.GpuOptions())
    done.append((tag, st.status.value, st.iterations, oob(tag)))


gm = load_golden("config0_s0")
run("config0 default", gm, eps_rel=1e-4)
for name, o in {"csr": dict(sell="off", row_order="natural"),
                "sell": dict(sell="on", sell_sort="off", row_order="natural"),
                "sell_sorted": dict(sell="on", sell_sort="on", row_order="natural"),
                "sell_rows": dict(sell="on", sell_sort="off", row_order="length", row_order_window=64),
                "csr_medium": dict(sell="off", medium_per_lane=1),
                "csr_split2": dict(sell="off", dual_split=2)}.items():
    run(f"config0 {name}", gm, eng.GpuOptions(**o), eps_rel=1e-12, max_kkt_passes=128)
c4 = config4(scale=0.002, seed=3)           # 10k x 20k, ~0.4M nnz
run("config4 0.2% rows", c4, eng.GpuOptions(row_order="length", sell="on"), eps_rel=1e-12, max_kkt_passes=130)
run("config4 0.2% csr", c4, eng.GpuOptions(sell="off", row_order="natural"), eps_rel=1e-12, max_kkt_passes=130)
c2 = config2(scale=0.002, seed=5)           # heavy-tailed rows -> block-per-row path
run("config2 0.2% heavy", c2, eng.GpuOptions(heavy_threshold=64), eps_rel=1e-12, max_kkt_passes=70)
dev = eng.device_lp(c4, eng.GpuOptions())
dev.spmv(np.ones(c4.n))
dev.spmv(np.ones(c4.m), transpose=True)
for kind, ov in (("loopback", "off"), ("loopback_fused", "off"), ("loopback", "on"), ("loopback", "serial")):
    pt, st = run_pdhg_sharded(gm, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=130), G=3, comm_kind=kind,
                              overlap=ov)
    done.append((f"sharded G=3 {kind} overlap={ov}", st.status.value, st.iterations, oob(kind)))
scaled, info = eng.ruiz_equilibrate(c4)
run("config4 0.2% after device Ruiz", scaled, eps_rel=1e-12, max_kkt_passes=64)
from paper_2603_03150_b200.instances import config1_general  # noqa: E402

g = config1_general(scale=0.002)
p, fmap = eng.to_standard_form(g)
s2, info2 = eng.ruiz_equilibrate(p)
pt, st = eng.run_pdhg(s2, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=64))
done.append(("config1 0.2% stdform+ruiz", st.status.value, st.iterations, oob("config1")))
from paper_2603_03150_b200 import finish  # noqa: E402

up = finish.unscale_point(info2, pt)
gp = finish.restrict_point(g, fmap, up)
vs = finish.violation_summary(p, up)
cs = finish.centered_start(up)
done.append(("finishing: unscale, restrict, violation, centered_start", float(vs.max_violation), len(gp[0])))
dev.spmv(np.ones(c4.n))
oob("spmv")
for d in done:
    print(d)
print(f"sanitize workload ok: {len(done)} runs; bounds-checked build: {CHECKED}; "
      f"out-of-bounds loads: {oob_total if CHECKED else 'n/a'}")
if CHECKED and oob_total:
    sys.exit(9)
