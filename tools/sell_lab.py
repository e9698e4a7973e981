"""Lab (not product): the product step kernels against minimal SpMV kernels
over the SAME sliced-ELL layouts of config 4 (tools/sell_lab.cu), rounds
interleaved in one process.

    python tools/sell_lab.py [--scale 1.0] [--rounds 5]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
LIB = ROOT / "tools" / "_libs" / "sell_lab.so"


def build():
    LIB.parent.mkdir(parents=True, exist_ok=True)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                    "-Xcompiler", "-fPIC", "-shared", str(ROOT / "tools" / "sell_lab.cu"), "-o", str(LIB)],
                   check=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    if not LIB.exists():
        build()
    import torch

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.engine import _start_vector
    from paper_2603_03150_b200.instances import config4

    lab = C.CDLL(str(LIB))
    lab.sell_lab_time.restype = C.c_int
    inst = config4(scale=args.scale, seed=4)
    d = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False))
    lam = d.opnorm(_start_vector(d.n, 0))
    st = 1.0 / (1.05 * lam)
    d.reset()
    dev = d.device
    g = torch.Generator(device="cpu").manual_seed(0)
    xn = torch.randn(d.n, generator=g, dtype=torch.float64).to(dev)
    xm = torch.randn(d.m, generator=g, dtype=torch.float64).to(dev)
    out = {"m": d.m, "n": d.n, "nnz": d.nnz, "heavy": list(d.heavy),
           "n_heavy": [int(d.a_heavy.numel()), int(d.at_heavy.numel())], "rounds": []}
    ops = {}
    for key, ptr, H, gx, rows in (("A", d.a_ptr, d.heavy[0], xn, d.m), ("At", d.at_ptr, d.heavy[1], xm, d.n)):
        s = d._sell[key]
        if s is None:
            raise SystemExit(f"{key} has no SELL layout")
        sd, (width, sp, scol, sval, perm) = s
        if perm is not None:
            out[f"{key}_note"] = "slice-sorted (perm): lab kernel ignores perm, rows are permuted within slices"
        y = torch.empty(rows, dtype=torch.float64, device=dev)
        v1 = torch.zeros(rows, dtype=torch.float64, device=dev)
        v2 = torch.zeros(rows, dtype=torch.float64, device=dev)
        bb = torch.ones(rows, dtype=torch.float64, device=dev)
        ops[key] = (sd, sp, width, scol, sval, ptr, H, gx, y, bb, v1, v2, rows)

    def lab_ms(key, kind, u):
        sd, sp, width, scol, sval, ptr, H, gx, y, bb, v1, v2, rows = ops[key]
        ms = C.c_float()
        rc = lab.sell_lab_time(kind, u, rows, sd.nslices, C.c_void_p(sp.data_ptr()), C.c_void_p(width.data_ptr()),
                               C.c_void_p(scol.data_ptr()), C.c_void_p(sval.data_ptr()), C.c_void_p(ptr.data_ptr()),
                               int(H), C.c_void_p(gx.data_ptr()), C.c_void_p(y.data_ptr()),
                               C.c_void_p(bb.data_ptr()), C.c_void_p(v1.data_ptr()), C.c_void_p(v2.data_ptr()),
                               args.reps, C.byref(ms))
        if rc:
            raise SystemExit(f"lab kernel error {rc}")
        return round(ms.value, 4)

    torch.cuda.synchronize()
    for r in range(args.rounds):
        row = {
            "product_dual": round(d.time_kernel(1, args.reps, st, st), 4),
            "lab_A_spmv_u10": lab_ms("A", 0, 10),
            "lab_A_spmv_u6": lab_ms("A", 0, 6),
            "lab_A_spmv_epi_u10": lab_ms("A", 1, 10),
            "lab_A_tail_10_2": lab_ms("A", 2, 10),
            "lab_A_tail_10_4": lab_ms("A", 3, 10),
            "lab_A_tail_8_2": lab_ms("A", 4, 10),
            "lab_A_tail_6_2": lab_ms("A", 5, 10),
            "product_primal": round(d.time_kernel(0, args.reps, st, st), 4),
            "lab_At_spmv_u6": lab_ms("At", 0, 6),
            "lab_At_spmv_u10": lab_ms("At", 0, 10),
            "lab_At_tail_6_2": lab_ms("At", 5, 10),
            "lab_At_tail_8_2": lab_ms("At", 4, 10),
            "clock": subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                                    capture_output=True, text=True).stdout.strip(),
        }
        out["rounds"].append(row)
        print(json.dumps(row), flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
