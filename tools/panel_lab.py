"""Lab (not product): band-panel SpMV (tools/panel_lab.cu) vs the product
SpMV on config 4's A (5M x 10M, 200M nnz) -- correctness and time.

    python tools/panel_lab.py [--scale 1.0] [--R 4096] [--W 14336] [--band 50000]

The layout is built on the GPU with torch: per entry (block b = row // R,
thread t = row % 1024, tag q = (row % R) // 1024); the block's band window is
[2*b*R - band, 2*(b+1)*R + band) (config 4: row i's band is centred on column
2i), cut into panels of W columns; entries outside go to the block's remote
list.  Keys (b, list, t, q, col) sorted once; slot = warp region + k*32 + lane.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
LIB = ROOT / "tools" / "_libs" / "panel_lab.so"
HEAVY = 256


def build_lib():
    LIB.parent.mkdir(parents=True, exist_ok=True)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                    "-Xcompiler", "-fPIC", "-shared", str(ROOT / "tools" / "panel_lab.cu"), "-o", str(LIB)],
                   check=True)


def layout(torch, A, R: int, W: int, band: int, dev):
    m, n = A.shape
    ptr = torch.from_numpy(A.indptr.astype("int64")).to(dev)
    col = torch.from_numpy(A.indices.astype("int64")).to(dev)
    val = torch.from_numpy(A.data).to(dev)
    nnz = col.numel()
    lens = ptr[1:] - ptr[:-1]
    row = torch.repeat_interleave(torch.arange(m, device=dev), lens)
    # rows renumbered by length (descending) inside each block, so a warp's
    # lanes hold rows of similar length; rows over `heavy` entries are left
    # out (the product runs them block per row)
    heavy = lens > HEAVY
    blk_of = torch.arange(m, device=dev) // R
    skey = blk_of * (1 << 20) + ((1 << 20) - 1 - torch.where(heavy, torch.zeros_like(lens), lens))
    newpos = torch.empty(m, dtype=torch.int64, device=dev)
    order_r = torch.sort(skey, stable=True).indices            # new position -> old row
    newpos[order_r] = torch.arange(m, device=dev)               # old row -> new position
    keep = ~heavy[row]
    row, col, val = row[keep], col[keep], val[keep]
    nnz = col.numel()
    b = newpos[row] // R
    r = newpos[row] % R
    t = r % 1024
    q = r // 1024
    nblk = (m + R - 1) // R
    wlo = (2 * torch.arange(nblk, device=dev) * R - band).clamp(min=0)
    wlo = wlo - (wlo % 2)
    whi = (2 * (torch.arange(nblk, device=dev) + 1) * R + band).clamp(max=n)
    npan = ((whi - wlo + W - 1) // W)                       # panels per block
    inb = (col >= wlo[b]) & (col < whi[b])
    lst = torch.where(inb, 1 + (col - wlo[b]) // W, torch.zeros_like(col))   # 0 = remote list
    maxl = int(npan.max()) + 1
    key = ((b * maxl + lst) * 1024 + t) * (R // 1024) + q
    key = key * (1 << 24) + col
    order = torch.sort(key, stable=True).indices
    del key
    b, lst, t, q, col, val, inb = (v[order] for v in (b, lst, t, q, col, val, inb))
    # rank of each entry inside its (b, list, t) group
    g = (b * maxl + lst) * 1024 + t
    first = torch.ones_like(g, dtype=torch.bool)
    first[1:] = g[1:] != g[:-1]
    idx = torch.arange(nnz, device=dev)
    start = torch.where(first, idx, torch.zeros_like(idx))
    start = torch.cummax(start, 0).values
    k = idx - start
    # panels that exist: per block the remote list + npan[b] panels (even empty ones)
    pan_count = npan + 1
    blk_pan = torch.zeros(nblk + 1, dtype=torch.int64, device=dev)
    blk_pan[1:] = torch.cumsum(pan_count, 0)
    npanels = int(blk_pan[-1])
    pid = blk_pan[b] + lst                                   # global panel id of each entry
    # width per (panel, warp) = 1 + max k over the warp's lanes
    warp = t // 32
    lane = t % 32
    wid = pid * 32 + warp
    width = torch.zeros(npanels * 32, dtype=torch.int64, device=dev)
    width.scatter_reduce_(0, wid, k + 1, reduce="amax")
    wslot = torch.zeros(npanels * 32, dtype=torch.int64, device=dev)
    wslot[1:] = torch.cumsum(32 * width, 0)[:-1]
    nslots = int((32 * width).sum())
    slot = wslot[wid] + k * 32 + lane
    sval = torch.zeros(nslots, dtype=torch.float64, device=dev)
    scq = torch.full((nslots,), -1, dtype=torch.int64, device=dev)
    sval[slot] = val
    pan_base_e = wlo[b] + (lst - 1) * W
    cq = torch.where(inb, (col - pan_base_e) | (q << 27), col | (q << 27))
    scq[slot] = cq
    scq32 = scq.to(torch.int64).bitwise_and(0xFFFFFFFF).to(torch.int32)   # bit pattern of the u32
    # per panel: base column and length (remote list: -1, 0)
    pb = torch.full((npanels,), -1, dtype=torch.int64, device=dev)
    pl = torch.zeros(npanels, dtype=torch.int64, device=dev)
    for_b = torch.repeat_interleave(torch.arange(nblk, device=dev), pan_count)
    lidx = torch.arange(npanels, device=dev) - blk_pan[:-1][for_b]
    base = wlo[for_b] + (lidx - 1) * W
    ln = torch.minimum(whi[for_b] - base, torch.full_like(base, W))
    ln = ln + (ln % 2)
    pb = torch.where(lidx > 0, base, pb)
    pl = torch.where(lidx > 0, ln, pl)
    stats = {"nslots": nslots, "nnz": nnz, "pad": nslots / nnz, "remote_frac": float((~inb).sum()) / nnz,
             "panels_per_block": float(npan.float().mean()), "nblk": nblk}
    stats["heavy_rows"] = int(heavy.sum())
    return dict(order_r=order_r, heavy=heavy, nblk=nblk, blk_pan=blk_pan.int(), pan_base=pb.int(), pan_len=pl.int(), wslot=wslot,
                wwidth=width.int(), val=sval, cq=scq32, stats=stats)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--R", type=int, default=4096)
    ap.add_argument("--W", type=int, default=14336)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--grid", type=int, default=148)
    args = ap.parse_args()
    build_lib()
    import numpy as np
    import torch

    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.instances import config4

    inst = config4(scale=args.scale, seed=4)
    band = max(int(50_000 * args.scale), 1)
    dev = torch.device("cuda", 0)
    t0 = time.time()
    L = layout(torch, inst.A, args.R, args.W, band, dev)
    torch.cuda.synchronize()
    print("layout", round(time.time() - t0, 1), "s", json.dumps(L["stats"]), flush=True)
    lib = C.CDLL(str(LIB))
    lib.panel_spmv.restype = C.c_int
    x = torch.from_numpy(np.random.default_rng(1).standard_normal(inst.n)).to(dev)
    y = torch.zeros(inst.m, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream()

    def call(mode=0):
        rc = lib.panel_spmv(L["nblk"], args.R, args.W, C.c_void_p(L["blk_pan"].data_ptr()),
                            C.c_void_p(L["pan_base"].data_ptr()), C.c_void_p(L["pan_len"].data_ptr()),
                            C.c_void_p(L["wslot"].data_ptr()), C.c_void_p(L["wwidth"].data_ptr()),
                            C.c_void_p(L["val"].data_ptr()), C.c_void_p(L["cq"].data_ptr()),
                            C.c_void_p(x.data_ptr()), inst.m, C.c_void_p(y.data_ptr()), args.grid,
                            C.c_void_p(s.cuda_stream), mode)
        assert rc == 0, rc

    call()
    torch.cuda.synchronize()
    A_light = inst.A.copy()
    hv = L["heavy"].cpu().numpy()
    ref = inst.A @ x.cpu().numpy()
    ref[hv] = 0.0                                   # heavy rows are not in the lab layout
    ref_new = ref[L["order_r"].cpu().numpy()]       # y is written in the renumbered order
    err = float(np.max(np.abs(y.cpu().numpy() - ref_new)) / max(1.0, np.max(np.abs(ref_new))))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    t_panel = e0.elapsed_time(e1) / args.reps
    modes = {}
    for mode, name in ((1, "no_tma"), (2, "no_remote"), (4, "no_panels"), (6, "tma_only"), (3, "panels_only_no_tma"),
                       (10, "panels_only_pipelined"), (8, "all_pipelined")):
        e0.record()
        for _ in range(args.reps):
            call(mode)
        e1.record()
        torch.cuda.synchronize()
        modes[name] = e0.elapsed_time(e1) / args.reps
    print("modes", json.dumps(modes), flush=True)
    # the product's SpMV of the same operator (renumbered rows + sliced ELL, and CSR-vector)
    out = {"panel_ms": t_panel, "panel_rel_err": err}
    for name, o in (("product_default", {}), ("product_csr", dict(sell="off", row_order="natural"))):
        d = eng.DeviceLp(inst.A, inst.b, inst.c, eng.GpuOptions(cache_layout=False, **o))
        vin = x
        outv = torch.empty(inst.m, dtype=torch.float64, device=dev)
        from paper_2603_03150_b200 import _native as N

        N.check(d.lib.pdhg_spmv(d.ctx, 0, vin.data_ptr(), outv.data_ptr()))
        torch.cuda.synchronize()
        e0.record(d.stream)
        for _ in range(args.reps):
            N.check(d.lib.pdhg_spmv(d.ctx, 0, vin.data_ptr(), outv.data_ptr()))
        e1.record(d.stream)
        torch.cuda.synchronize()
        out[name + "_ms"] = e0.elapsed_time(e1) / args.reps
        del d
        torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
