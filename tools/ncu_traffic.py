"""Summarise an ncu --set full capture of the step kernels into
profiles/traffic.json (read by bench.py for roofline.traffic and the binding
units).  Runs here, on the .ncu-rep brought back from the GPU box:

    python tools/ncu_traffic.py gpurun_out/X_full.ncu-rep [--source "command ..."]
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import re
import statistics
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

UNITS = {
    "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex2xbar_req_pct": "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}


def _num(v: str) -> float:
    return float(v.replace(",", "")) if v not in ("", "n/a") else float("nan")


def load(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        d["_units"] = dict(zip(head, units))
        res.append(d)
    return res


def scale(d: dict, key: str) -> float:
    """Metric value in base units (bytes, us, GHz) whatever ncu's display unit."""
    v, u = _num(d[key]), d["_units"].get(key, "")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
            "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3,
            "Ghz": 1.0, "GHz": 1.0, "Mhz": 1e-3, "MHz": 1e-3, "hz": 1e-9, "cycle/nsecond": 1.0,
            "cycle/usecond": 1e-3}.get(u, 1.0)
    return v * mult


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--source", default="")
    ap.add_argument("--out", default=str(ROOT / "profiles" / "traffic.json"))
    args = ap.parse_args()
    launches = load(args.rep)
    groups: dict[str, list[dict]] = {"primal": [], "dual": []}
    names = {}
    for d in launches:
        name = d.get("Kernel Name", "")
        # the ordinary step kernels only (not the check-fused last iteration's
        # k_step_sell_chk / quad-writing k_step_sell<1, U, 1>)
        m = re.search(r"(k_step(?:_sell)?)<(\w+)(?:, (\w+))?(?:, (\w+))?>", name)
        if not m or m.group(4) == "1":
            continue
        key = "primal" if m.group(2) in ("1", "true") else "dual"
        groups[key].append(d)
        names[key] = name
    out = {}
    for key, ds in groups.items():
        if not ds:
            continue
        traffic = [scale(d, "dram__bytes_read.sum") + scale(d, "dram__bytes_write.sum") for d in ds]
        out[key] = int(statistics.median(traffic))
        u = {k: round(statistics.median(_num(d[m]) for d in ds), 6) for k, m in UNITS.items()}
        u["time_us"] = round(statistics.median(scale(d, "gpu__time_duration.sum") for d in ds), 3)
        u["sm_ghz"] = round(statistics.median(scale(d, "sm__cycles_elapsed.avg.per_second") for d in ds), 3)
        u["launches"] = len(ds)
        u["kernel"] = names[key]
        out[f"{key}_units"] = u
    out["_source"] = args.source or f"{args.rep}: dram__bytes_read.sum + dram__bytes_write.sum per launch (median)"
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
