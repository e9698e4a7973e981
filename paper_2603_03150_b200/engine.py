"""Host side of the B200 PDHG engine: the reference's `run_pdhg` control flow
over the sm_100a kernels of libpdhg_b200.so.

Drop-in for ``hybridlp.pdhg.run_pdhg`` (/root/reference/pkg/src/hybridlp/
pdhg.py:162-258): same signature, same options object, same result objects,
same status/raise behaviour.  The loop below follows the reference line by
line, at the granularity of one *period* (the iterations up to the next KKT
check, pdhg.py:198-199): the device runs a whole period as one CUDA graph and
returns ~16 scalars; every decision (termination, candidate, best point,
restart, primal weight) is taken here from those scalars exactly as the
reference takes it.

Differences from the reference, all documented in DESIGN.md:
  * the time limit is tested before every period instead of every step
    (pdhg.py:188); time_limit_s=0 still returns after 0 iterations;
  * sums (SpMV rows, norms, dots) run in a different but fixed order, so
    scores agree to rounding (1e-16 relative), not bit for bit.
"""

from __future__ import annotations

import ctypes as C
import dataclasses
import math
import threading
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from . import hostio, streams
from .lp_types import resolve

_WEIGHT_CLIP = (1e-4, 1e4)  # pdhg.py:28


@dataclass
class GpuOptions:
    """GPU-only knobs (keyword-only in run_pdhg, never required).

    device:          CUDA device index (default: current device).
    a_lanes/at_lanes: lanes per row for A / A' rows (0 = auto from the mean row length).
    heavy_threshold: rows longer than this get a whole thread block (0 = auto per
                     operator: 32 x lanes per row, so a light warp never runs more
                     than ~8 dependent load rounds on one row; measured on config 1,
                     profiles/r01_pipeline.md).
    medium_per_lane: CSR step kernels: rows longer than this many entries per lane
                     (x lanes per row) but not heavy run one warp per row, so a
                     long row does not hold a warp-owns-32-rows pass for many
                     dependent load rounds.  -1 = auto: 8 for <= 8 lanes per row
                     (config 1's dual step 12.1 -> 9.8 us), 16 for 16 lanes (config
                     2's 104.6 -> 99.4 us; 8 would slow config 4's 944 -> 976 us);
                     0 = off.
    opnorm:          override the power-iteration estimate (parity fallback).
    cache_layout:    keep the device layout of a model for repeated solves.
    psr:             "auto" | "on" | "off" -- panel-staged rows layout for the step
                     kernels (csrc/psr.cuh); auto uses it when >= psr_min_fraction of
                     the entries fall in staged panels and the operator has enough rows.
    psr_min_staged:  entries a (row block, panel) needs to be staged in shared memory.
    dual_split:      column chunks of the dual step's SpMV (split-K, csrc k_dual_split):
                     each pass gathers from an L2-sized window of xe; 1 = unsplit.
    sell:            "auto" | "on" | "off" -- sliced-ELL layout (csrc/sell_build.cu) for
                     the step kernels; auto uses it for an operator whose padded slot
                     count stays within sell_max_pad x its nonzeros (near-uniform row
                     lengths), that has no PSR layout, and either short rows (mean <
                     sell_max_mean: config 3, steps 10-22 % faster) or >= sell_min_nnz
                     entries (with 6 entries in flight per lane: config 4's A' primal
                     step 0.862 -> 0.780 ms, config 2's A' (18M) 81.6 -> 73.6 us,
                     config 4 at 5 % (10M) 41.3 -> 35.6 us; at 1.5M entries it measured
                     50 % slower).  Skewed rows (config 4's A: 4x padding) stay on
                     CSR-vector.
    row_order:       "auto" | "length" | "natural" -- "length" renumbers the rows of A
                     (the constraints: b, y) by decreasing length inside windows of
                     row_order_window rows on the device, so consecutive rows -- one
                     sliced-ELL slice -- have equal lengths and the dual step runs on
                     sliced ELL without padding (config 4's A: 4.1x padded in natural
                     order, ~1.03x renumbered).  y is mapped back on every
                     download, so results are the same LP's.  auto: unsharded operators
                     with >= sell_min_nnz entries whose natural-order padding exceeds
                     sell_max_pad and at most row_order_max_tail of whose entries sit
                     in rows longer than 4x the mean (lane-per-row slices run a long
                     row on one lane: config 2's power-law rows stay on CSR-vector).
    col_order:       "auto" | "length" | "natural" -- the same for A's columns (the
                     variables: c, x, z; the rows of A'), so the primal step's sliced
                     ELL of A' runs without padding (config 4's A': 1.49x slice-sorted
                     in natural order; -4.4 % per primal SpMV at the power cap,
                     tools/primal_pad_lab.cu).  A's entries keep their order inside
                     each row (only their column labels change) and A' rows keep
                     theirs, so every step's sums are the unrenumbered ones; x and z
                     are mapped back on download.  auto: whenever row_order applies.
    col_order_first: columns longer than this come first (as row_order_first).
    row_order_window: rows (and columns) per renumbering window: 16k measured best
                     on config 4 (per period, rotated A/B: 16k 112.7, 32k 113.0,
                     8k 113.1, 64k 113.9, 256k 115.6 ms; profiles/r02_ab_window*.log).
    row_order_first: with row_order: rows longer than this many entries come first
                     (window by window, longest first), then the rest -- the long
                     slices start at the head of the grid, so no window's long slices
                     are left running after the rest has drained (config 4's dual
                     SpMV 0.889 -> 0.789 ms, tools/rowlen_lab.cu).  0 = plain windows;
                     -1 = every log2 length class in turn, longest first.
    sell_sort:       "auto" | "on" | "off" -- order each slice's rows by length (lanes
                     active in a round form a prefix, so fetched sectors are full):
                     config 4's A' reads 3.55 instead of 3.85 GB per primal step (period
                     ~0.5 % faster); config 3's 1-3 entry rows lose to the extra dependent
                     load per warp, so auto sorts operators with mean row length >= 12.
    persistent:      "off" | "on" | "tiny" | "auto" -- "off" (default): a CUDA graph of two
                     kernels per iteration; "on": each period as one cooperative kernel
                     (grid barriers between half steps); "tiny": each period as one
                     single-block kernel (model in one SM's L1); "auto": tiny for
                     nnz <= tiny_max_nnz and m + n <= tiny_max_rows.  Both persistent
                     forms are parity-tested and measured no faster than the graph
                     (profiles/r01_pipeline.md); CSR layouts, unsharded.
    l2_persist:      bit mask: 1 = pin y in L2 for the primal step, 2 = pin xe for the
                     dual step (persisting access-policy window; L2 holds 79 MB persisting).
    check_dot:       reuse A'y of the checked points (both computed by the two-point
                     check) as the SpMV of the next period's first primal step
                     (pdhg_use_check_dot; bit-identical iterates).  Applies when A' has a
                     sliced-ELL layout, unsharded: config 4 skips one of the 64 primal
                     SpMVs of every period.
    check_fuse:      run the two-point check's A side inside the last iteration of each
                     period (pdhg_check_fuse_enable): one pass over A gives the dual step's
                     A xe and the check's A x, A avg_x from (xe, x, avg_x) quads; bitwise
                     the same iterates and check scalars.  Applies when A and A' both have
                     sliced-ELL layouts, unsharded (config 4).
    split_full_sell: shards with split steps (overlapped multi-GPU schedule) also lay
                     out their whole rows in sliced ELL (when the padding gate passes),
                     for the two-point check and the power iteration; the split steps
                     run over their own part layouts either way.
    """

    device: int | None = None
    a_lanes: int = 0
    at_lanes: int = 0
    heavy_threshold: int = 0
    medium_per_lane: int = -1
    opnorm: float | None = None
    cache_layout: bool = True
    psr: str = "off"
    psr_min_staged: int = 1024
    psr_min_fraction: float = 0.3
    psr_min_rows: int = 148 * 256
    l2_persist: int = 0
    dual_split: int = 1
    persistent: str = "off"
    graphs: bool = True
    tiny_max_nnz: int = 200_000
    tiny_max_rows: int = 65_536
    sell: str = "auto"
    sell_max_pad: float = 1.6
    sell_max_mean: float = 12.0
    sell_min_nnz: int = 5_000_000
    sell_sort: str = "auto"
    row_order: str = "auto"
    row_order_window: int = 16384
    row_order_max_tail: float = 0.15
    row_order_first: int = 32
    col_order: str = "auto"
    col_order_first: int = 32
    check_dot: bool = True
    check_fuse: bool = True
    split_full_sell: bool = True


def auto_lanes(nnz: int, rows: int) -> int:
    """Lanes per row from the mean row length (csrc auto_lanes; measured on
    config 4, profiles/r01_spmv_lab2.log)."""
    if rows <= 0:
        return 1
    mean = nnz / rows
    for lanes, lo in ((32, 80), (16, 32), (8, 12), (4, 6), (2, 3)):
        if mean >= lo:
            return lanes
    return 1


def heavy_threshold(lanes: int) -> int:
    """Auto heavy-row threshold for an operator processed with `lanes` lanes per row.

    Rows between 8-16 entries per lane and this threshold run warp-per-row
    (the medium tier), so only rows of >= 128 entries need a whole block:
    config 1 (2 lanes) dual step 10.5 -> 8.7 us with 128 instead of 64;
    16 lanes keeps 512 (1,024 measured 7 % slower on config 2)."""
    return max(128, 32 * lanes)


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise N.NativeError("paper_2603_03150_b200 needs a CUDA device (B200, sm_100a); "
                            "there is no CPU fallback")
    return torch


def _medium_list(torch, ptr, lanes: int, H: int, per_lane: int):
    """Rows with per_lane*lanes < length <= H (row order) and that light limit."""
    if per_lane < 0:
        per_lane = 8 if lanes <= 8 else 16
    light_max = per_lane * lanes
    if per_lane <= 0 or lanes >= 32 or light_max >= H:
        return torch.empty(0, dtype=torch.int32, device=ptr.device), 0
    lens = ptr[1:] - ptr[:-1]
    idx = torch.nonzero((lens > light_max) & (lens <= H)).flatten().to(torch.int32).contiguous()
    return idx, light_max


def _slice_pad(torch, ptr, H: int) -> float:
    """Padded slots / entries of the natural-order sliced ELL of a CSR operator
    (rows longer than H excluded, as the SELL plan does)."""
    lens = (ptr[1:] - ptr[:-1]).to(torch.int64)
    lens = torch.where(lens > H, torch.zeros_like(lens), lens)
    rows = lens.numel()
    pad_rows = (-rows) % 32
    if pad_rows:
        lens = torch.cat([lens, torch.zeros(pad_rows, dtype=lens.dtype, device=lens.device)])
    slots = 32 * int(lens.view(-1, 32).max(dim=1).values.sum())
    return slots / max(1, int(lens.sum()))


def _want_row_order(torch, opts, ptr, nnz: int, H: int) -> bool:
    if opts.row_order == "length":
        return True
    if opts.row_order != "auto" or opts.sell == "off" or opts.psr != "off" or nnz < opts.sell_min_nnz:
        return False
    if opts.persistent not in ("off", "auto") or int(opts.dual_split) > 1:
        return False
    # heavy-tailed operators stay on CSR-vector: lane-per-row sliced ELL runs a
    # long row on one lane (config 2's power-law A, 52 % of its entries in rows
    # over 4x the mean: 10.1 -> 15.3 s to 1e-4 renumbered); config 4's
    # lognormal A has 9 % there
    lens = (ptr[1:] - ptr[:-1]).to(torch.int64)
    mean = float(nnz) / max(1, lens.numel())
    tail = float(lens[lens > 4 * mean].sum()) / max(1, nnz)
    if tail > opts.row_order_max_tail:
        return False
    return _slice_pad(torch, ptr, H) > opts.sell_max_pad


def _length_order(torch, dev, lens, window: int, first: int):
    """New -> old index order of a row renumbering: decreasing length inside
    windows of `window` rows (stable); with first > 0 the rows longer than
    `first` come first (window by window), then the rest -- their slices start
    at the head of the grid instead of at every window's head, where the last
    windows' long slices were still running after everything else had drained
    (config 4's dual step: 0.889 -> 0.789-0.795 ms, tools/rowlen_lab.cu);
    first < 0: every log2 length class in turn, longest first."""
    k = lens.numel()
    top = int(lens.max()) + 1 if k else 1
    win = torch.arange(k, device=dev, dtype=torch.int64) // max(1, window)
    key = win * (top + 1) + (top - lens)
    first = int(first)
    if first != 0 and k:
        if first > 0:
            group = (lens <= first).to(torch.int64)            # 0: longer than `first`
        else:
            cls = torch.floor(torch.log2(lens.clamp(min=1).to(torch.float64))).to(torch.int64)
            group = int(cls.max()) - cls
        key = group * (int(win.max()) + 1) * (top + 1) + key
    return torch.sort(key, stable=True).indices


def _close_ctx(lib, ctx, stream) -> None:
    """DeviceLp finalizer: destroy the context; a pooled stream is drained
    (its queued work may still read this layout, whose blocks are about to go
    back to the allocator) and returned to the pool."""
    if stream is not None:
        stream.synchronize()
    lib.pdhg_ctx_destroy(ctx)
    if stream is not None:
        streams.release(stream)


def _as_csr(A):
    import scipy.sparse as sp

    if not sp.isspmatrix_csr(A) and not isinstance(A, sp.csr_array):
        A = sp.csr_matrix(A, dtype=float)
    if A.dtype != np.float64:
        A = A.astype(np.float64)
    return A


class DeviceLp:
    """Device-resident dual layout of one StandardLp plus the engine context.

    Owns (as torch tensors) A in CSR, A' in CSR (built on the device, equal to
    scipy's tocsc arrays), b, c, the heavy-row lists and the workspace the
    library carves its iterate buffers from.
    """

    def __init__(self, A, b, c, opts: GpuOptions, *, shard=None, stream=None, device_arrays=None,
                 ws_alloc=None):
        """``shard`` (sharded.ShardBlock) makes this the context of one shard:
        A is then the shard's row block with column indices in padded
        x-space slots, ``shard.At`` its block of A' rows (CSR, y-space
        slots), and the iterate vectors have the padded full lengths.
        ``stream``: a torch.cuda.Stream to share (loopback shards).
        ``device_arrays``: (indptr, indices, data) of A already on the device
        (e.g. the output of the device Ruiz pass) -- not uploaded again.
        ``ws_alloc``: allocator (nbytes, device) -> uint8 tensor for the iterate
        workspace (symmetric memory for the fused multi-GPU all-gather)."""
        torch = _torch()
        t_start = time.monotonic()
        self.lib = N.load()
        dev = torch.device("cuda", torch.cuda.current_device() if opts.device is None else opts.device)
        self.device = dev
        self.lock = threading.Lock()
        A = _as_csr(A)
        m, n = A.shape
        nnz = int(A.nnz)
        if nnz >= 2**31 - 1:
            raise ValueError("nnz >= 2^31 is not supported by the int32 layout")
        if shard is not None:
            At = _as_csr(shard.At)
            n = At.shape[0]                       # rows of A' this shard owns
            m_full, n_full = shard.m_full, shard.n_full
            y_off, x_off = shard.y_off, shard.x_off
            if A.shape[1] != n_full or At.shape[1] != m_full:
                raise ValueError("inconsistent shard block shapes")
        else:
            At = None
            m_full, n_full, y_off, x_off = m, n, 0, 0
        self.m, self.n, self.nnz = m, n, nnz
        self.at_nnz = int(At.nnz) if At is not None else nnz
        self.m_full, self.n_full, self.y_off, self.x_off = m_full, n_full, y_off, x_off
        with torch.cuda.device(dev):
            # pooled: the next context on this device reuses the stream and so the
            # caching allocator's blocks of this one (paper_2603_03150_b200/streams.py)
            self.stream = stream if stream is not None else streams.acquire(dev)
            own_stream = stream is None
            with torch.cuda.stream(self.stream):
                t = lambda a, dt: hostio.h2d(a, dt, dev)
                if device_arrays is not None:
                    self.a_ptr, self.a_col, self.a_val = device_arrays
                else:
                    self.a_ptr = t(A.indptr, np.int32)
                    self.a_col = t(A.indices, np.int32)
                    self.a_val = t(A.data, np.float64)
                self.b = t(b, np.float64)
                self.c = t(c, np.float64)
                self.stream.synchronize()
                t_up = time.monotonic()
                self.row_perm = self.row_inv = None
                self.col_perm = self.col_inv = None
                self._col_perm_host = None
                t_rs = t_rn = t_up
                if shard is None:
                    want = False
                    if m > 1:
                        lanes0 = int(opts.a_lanes) or auto_lanes(nnz, m)
                        H0 = int(opts.heavy_threshold) or heavy_threshold(lanes0)
                        want = _want_row_order(torch, opts, self.a_ptr, nnz, H0)
                    t_rs = t_rn = time.monotonic()
                    if want:
                        self._renumber_rows(torch, dev, m, nnz, int(opts.row_order_window),
                                            int(opts.row_order_first))
                    if n > 1 and (opts.col_order == "length" or (opts.col_order == "auto" and want)):
                        self._renumber_cols(torch, dev, n, nnz, int(opts.row_order_window),
                                            int(opts.col_order_first))
                    t_rn = time.monotonic()
                sptr = self.stream.cuda_stream
                tmp = None
                if At is None:
                    self.at_ptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
                    self.at_col = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
                    self.at_val = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
                    tmp_bytes = self.lib.pdhg_transpose_tmp_bytes(nnz, m, n)
                    tmp = torch.empty(max(tmp_bytes, 1), dtype=torch.uint8, device=dev)
                    N.check(self.lib.pdhg_transpose_csr(
                        m, n, nnz, self.a_ptr.data_ptr(), self.a_col.data_ptr(), self.a_val.data_ptr(),
                        self.at_ptr.data_ptr(), self.at_col.data_ptr(), self.at_val.data_ptr(),
                        tmp.data_ptr(), tmp_bytes, sptr))
                else:
                    self.at_ptr = t(At.indptr, np.int32)
                    self.at_col = t(At.indices, np.int32)
                    self.at_val = t(At.data, np.float64)
                self.stream.synchronize()
                t_tr = time.monotonic()
                t_tr0 = t_rn
                self.a_lanes = int(opts.a_lanes) or auto_lanes(nnz, m)
                self.at_lanes = int(opts.at_lanes) or auto_lanes(self.at_nnz, n)
                H = int(opts.heavy_threshold) or heavy_threshold(self.a_lanes)
                Ht = int(opts.heavy_threshold) or heavy_threshold(self.at_lanes)
                self.heavy = (H, Ht)
                self.a_heavy = torch.nonzero((self.a_ptr[1:] - self.a_ptr[:-1]) > H).flatten().to(torch.int32)
                self.at_heavy = torch.nonzero((self.at_ptr[1:] - self.at_ptr[:-1]) > Ht).flatten().to(torch.int32)
                self.a_medium, la = _medium_list(torch, self.a_ptr, self.a_lanes, H, opts.medium_per_lane)
                self.at_medium, lt = _medium_list(torch, self.at_ptr, self.at_lanes, Ht, opts.medium_per_lane)
                t_lists = time.monotonic()
                self.light_max = (la, lt)
                self.psr_info = {}
                self._psr = {}
                for key, rows, cols, nz, ptr, col, val in (
                        ("A", m, n_full, nnz, self.a_ptr, self.a_col, self.a_val),
                        ("At", n, m_full, self.at_nnz, self.at_ptr, self.at_col, self.at_val)):
                    self._psr[key] = self._build_psr(torch, dev, key, rows, cols, nz, ptr, col, val,
                                                     H if key == "A" else Ht, opts)
                pers = opts.persistent
                if pers == "auto":
                    pers = ("tiny" if nnz <= opts.tiny_max_nnz and m + n <= opts.tiny_max_rows
                            and shard is None and opts.psr == "off" and int(opts.dual_split) <= 1
                            and N.experimental() else "off")
                if (pers in ("on", "tiny") or int(opts.l2_persist) & 3) and not N.experimental():
                    raise N.NativeError(f"persistent={pers!r} / l2_persist need the experiment build of "
                                        "libpdhg_b200 (both measured slower; python -m "
                                        "paper_2603_03150_b200.build --experimental)")
                self.persistent_mode = pers
                self._sell = {}
                self.sell_info = {}
                # split steps (sharded local-first blocks, overlapped schedule): pass 0 =
                # each row's local-slot entries, pass 1 = the rest + epilogue (CSR kernels)
                self.split_local = {"A": None, "At": None}
                if shard is not None and getattr(shard, "a_nloc", None) is not None:
                    for key, ptr, nloc in (("A", self.a_ptr, shard.a_nloc), ("At", self.at_ptr, shard.at_nloc)):
                        nl = torch.from_numpy(np.ascontiguousarray(nloc, dtype=np.int32)).to(dev)
                        self.split_local[key] = (ptr[:-1] + nl).contiguous()
                for key, rows, nz, ptr, col, val, Hk in (
                        ("A", m, nnz, self.a_ptr, self.a_col, self.a_val, H),
                        ("At", n, self.at_nnz, self.at_ptr, self.at_col, self.at_val, Ht)):
                    self._sell[key] = None if (self._psr[key] or pers in ("tiny", "on")
                                               or (self.split_local[key] is not None
                                                   and not opts.split_full_sell)) else \
                        self._build_sell(torch, dev, key, rows, nz, ptr, col, val, Hk, opts)
                # split steps (overlapped multi-GPU schedule) over sliced-ELL parts:
                # part 0 = each row's local-slot entries, part 1 = the rest
                self._sell_part = {"A": None, "At": None}
                for key, rows, ptr, col, val, Hk in (
                        ("A", m, self.a_ptr, self.a_col, self.a_val, H),
                        ("At", n, self.at_ptr, self.at_col, self.at_val, Ht)):
                    if self.split_local[key] is not None and opts.sell != "off" and rows > 0:
                        self._sell_part[key] = self._build_sell_parts(torch, dev, key, rows, ptr, col, val,
                                                                      self.split_local[key], Hk, opts)
                self.stream.synchronize()
                t_sell = time.monotonic()
                self.a_split = None
                self.nsplit = 1
                K = int(opts.dual_split)
                if K > 1 and n_full >= 4 * K and m * (K - 1) < 2**31:
                    chunk = (n_full + K - 1) // K
                    split = torch.empty((K - 1) * m, dtype=torch.int32, device=dev)
                    flag = torch.empty(1, dtype=torch.int32, device=dev)
                    uns = C.c_int32()
                    N.check(self.lib.pdhg_split_build(m, self.a_ptr.data_ptr(), self.a_col.data_ptr(), K,
                                                      chunk, split.data_ptr(), flag.data_ptr(), sptr,
                                                      C.byref(uns)))
                    if not uns.value:
                        self.a_split, self.nsplit = split, K
                ws_bytes = self.lib.pdhg_workspace_bytes(m_full, n_full)
                self.ws = (ws_alloc(ws_bytes, dev) if ws_alloc is not None
                           else torch.empty(ws_bytes, dtype=torch.uint8, device=dev))
                self.stream.synchronize()
                del tmp
        p = N.Problem()
        p.m, p.n, p.nnz = m, n, nnz
        p.a_ptr, p.a_col, p.a_val = self.a_ptr.data_ptr(), self.a_col.data_ptr(), self.a_val.data_ptr()
        p.at_ptr, p.at_col, p.at_val = self.at_ptr.data_ptr(), self.at_col.data_ptr(), self.at_val.data_ptr()
        p.b, p.c = self.b.data_ptr(), self.c.data_ptr()
        p.a_lanes, p.at_lanes, p.heavy_threshold = self.a_lanes, self.at_lanes, H
        p.at_heavy_threshold = Ht
        p.persistent = {"on": 1, "tiny": 2}.get(self.persistent_mode, 0 if opts.graphs else 3)
        p.a_sell = C.pointer(self._sell["A"][0]) if self._sell["A"] else None
        p.at_sell = C.pointer(self._sell["At"][0]) if self._sell["At"] else None
        p.a_n_heavy, p.at_n_heavy = self.a_heavy.numel(), self.at_heavy.numel()
        p.a_light_max, p.at_light_max = self.light_max
        p.a_n_medium, p.at_n_medium = self.a_medium.numel(), self.at_medium.numel()
        p.a_medium = self.a_medium.data_ptr() if p.a_n_medium else None
        p.at_medium = self.at_medium.data_ptr() if p.at_n_medium else None
        p.a_heavy = self.a_heavy.data_ptr() if p.a_n_heavy else None
        p.at_heavy = self.at_heavy.data_ptr() if p.at_n_heavy else None
        p.a_psr = C.pointer(self._psr["A"][0]) if self._psr["A"] else None
        p.at_psr = C.pointer(self._psr["At"][0]) if self._psr["At"] else None
        p.l2_persist = int(opts.l2_persist) & 3
        p.m_full, p.n_full, p.y_off, p.x_off = m_full, n_full, y_off, x_off
        p.at_nnz = self.at_nnz
        p.a_nsplit = self.nsplit
        p.a_split = self.a_split.data_ptr() if self.a_split is not None else None
        if self.split_local["A"] is not None:
            p.a_nsplit, p.a_split = 2, self.split_local["A"].data_ptr()
        if self.split_local["At"] is not None:
            p.at_nsplit, p.at_split = 2, self.split_local["At"].data_ptr()
        for key, fs, fp in (("A", "a_sell_part", "a_part_ptr"), ("At", "at_sell_part", "at_part_ptr")):
            parts = self._sell_part.get(key)
            if parts is not None:
                sells, keep = parts
                for h in range(2):
                    getattr(p, fs)[h] = C.addressof(sells[h])
                    getattr(p, fp)[h] = keep[h][0].data_ptr()
        self._prob = p
        ctx = C.c_void_p()
        N.check(self.lib.pdhg_ctx_create(C.byref(p), self.ws.data_ptr(), ws_bytes,
                                         self.stream.cuda_stream, C.byref(ctx)))
        self.ctx = ctx
        # check -> first primal step reuse (sliced ELL of A', one GPU)
        self.check_dot = bool(opts.check_dot and shard is None and p.at_sell
                              and self.lib.pdhg_check_dot_enable(ctx, 1) == 0)
        # two-point check's A side fused into each period's last dual step
        self.check_fuse = bool(opts.check_fuse and shard is None and p.a_sell and p.at_sell
                               and self.lib.pdhg_check_fuse_enable(ctx, 1) == 0)
        t_end = time.monotonic()
        self.timings = {"upload_s": t_up - t_start, "layout_s": t_end - t_up,
                        "layout_detail": {"row_order_choice_s": t_rs - t_up, "renumber_s": t_rn - t_rs,
                                          "transpose_s": t_tr - t_tr0, "row_lists_s": t_lists - t_tr,
                                          "psr_sell_s": t_sell - t_lists, "ctx_s": t_end - t_sell}}
        self._fin = weakref.finalize(self, _close_ctx, self.lib, ctx, self.stream if own_stream else None)
        self._scal = (C.c_double * (2 * N.NQ))()

    def _renumber_rows(self, torch, dev, m: int, nnz: int, window: int, first: int = 0):
        """Renumber A's rows by decreasing length inside windows of `window` rows
        (stable): new row r = old row row_perm[r].  A, b are permuted on the
        device; y-space results are mapped back through row_inv."""
        lens = (self.a_ptr[1:] - self.a_ptr[:-1]).to(torch.int64)
        perm = _length_order(torch, dev, lens, window, first)
        new_ptr = torch.zeros(m + 1, dtype=torch.int32, device=dev)
        new_ptr[1:] = torch.cumsum(lens[perm], 0).to(torch.int32)
        new_col = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        new_val = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        perm32 = perm.to(torch.int32)
        N.check(self.lib.pdhg_permute_rows(m, perm32.data_ptr(), self.a_ptr.data_ptr(), self.a_col.data_ptr(),
                                           self.a_val.data_ptr(), new_ptr.data_ptr(), new_col.data_ptr(),
                                           new_val.data_ptr(), self.stream.cuda_stream))
        self.b = self.b[perm].contiguous()
        inv = torch.empty_like(perm)
        inv[perm] = torch.arange(m, device=dev, dtype=torch.int64)
        self.stream.synchronize()
        self.a_ptr, self.a_col, self.a_val = new_ptr, new_col, new_val
        self.row_perm, self.row_inv = perm, inv
        self._row_perm_host = None      # host copy made on first use (spmv gates only)

    def _renumber_cols(self, torch, dev, n: int, nnz: int, window: int, first: int = 0):
        """Renumber A's columns (the rows of A', built next by the transpose) by
        decreasing length, as _renumber_rows does for A's rows: new column j =
        old column col_perm[j].  A's entries are relabelled in place of order
        (each row keeps its entry sequence), c is permuted; x-space results
        are mapped back through col_inv."""
        col = self.a_col[:nnz]
        lens = torch.bincount(col, minlength=n).to(torch.int64)
        perm = _length_order(torch, dev, lens, window, first)
        inv = torch.empty_like(perm)
        inv[perm] = torch.arange(n, device=dev, dtype=torch.int64)
        inv32 = inv.to(torch.int32)
        new_col = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        torch.index_select(inv32, 0, col, out=new_col[:nnz])
        self.c = self.c[perm].contiguous()
        self.stream.synchronize()
        self.a_col = new_col
        self.col_perm, self.col_inv = perm, inv

    def _build_sell(self, torch, dev, key, rows, nnz, ptr, col, val, H, opts):
        """Plan + fill the sliced-ELL layout of one operator on the device (or None)."""
        if opts.sell == "off" or rows <= 0 or nnz <= 0:
            return None
        if opts.sell == "auto" and nnz / rows >= opts.sell_max_mean and nnz < opts.sell_min_nnz:
            return None
        lib = self.lib
        sptr_ = self.stream.cuda_stream
        ns = (rows + 31) // 32
        width = torch.empty(ns, dtype=torch.int32, device=dev)
        sp = torch.empty(ns + 1, dtype=torch.int64, device=dev)
        tb = lib.pdhg_sell_tmp_bytes(rows)
        tmp = torch.empty(max(tb, 1), dtype=torch.uint8, device=dev)
        slots = C.c_int64()
        N.check(lib.pdhg_sell_plan(rows, ptr.data_ptr(), int(H), width.data_ptr(), sp.data_ptr(),
                                   tmp.data_ptr(), tb, sptr_, C.byref(slots)))
        pad = slots.value / max(1, nnz)
        self.sell_info[key] = {"slots": slots.value, "pad": pad, "used": False}
        if opts.sell == "auto" and pad > opts.sell_max_pad:
            return None
        scol = torch.empty(max(slots.value, 1), dtype=torch.int32, device=dev)
        sval = torch.empty(max(slots.value, 1), dtype=torch.float64, device=dev)
        perm = inv = None
        sort = opts.sell_sort if isinstance(opts.sell_sort, str) else ("on" if opts.sell_sort else "off")
        if (key == "A" and self.row_perm is not None) or (key == "At" and self.col_perm is not None):
            sort = "off"     # already ordered by length (row_order / col_order)
        if sort == "on" or (sort == "auto" and nnz / rows >= 12):
            perm = torch.empty(ns * 32, dtype=torch.uint8, device=dev)
            inv = torch.empty(ns * 32, dtype=torch.uint8, device=dev)
            N.check(lib.pdhg_sell_sort(rows, ptr.data_ptr(), int(H), perm.data_ptr(), inv.data_ptr(), sptr_))
        N.check(lib.pdhg_sell_fill(rows, ptr.data_ptr(), col.data_ptr(), val.data_ptr(), int(H),
                                   sp.data_ptr(), inv.data_ptr() if inv is not None else None,
                                   scol.data_ptr(), sval.data_ptr(), sptr_))
        d = N.Sell()
        d.rows, d.nslices = rows, ns
        d.sptr, d.width, d.col, d.val = sp.data_ptr(), width.data_ptr(), scol.data_ptr(), sval.data_ptr()
        d.perm = perm.data_ptr() if perm is not None else None
        d.nslots = slots.value
        self.stream.synchronize()
        del inv
        self.sell_info[key]["used"] = True
        self.sell_info[key]["sorted"] = perm is not None
        return (d, (width, sp, scol, sval, perm))

    def _build_sell_parts(self, torch, dev, key, rows, ptr, col, val, split, H, opts):
        """Sliced-ELL layouts of the two passes of a split step: each row's
        entries [ptr, split) and [split, ptr+1) as two CSR matrices on the
        device, heavy rows (> H entries, run whole in pass 1) left out of
        both, each laid out by _build_sell.  -> ([Sell, Sell], keep-alive), or
        None when either part's sliced ELL is rejected (slice padding beyond
        sell_max_pad under sell="auto")."""
        i64 = torch.int64
        full = (ptr[1:] - ptr[:-1]).to(i64)
        light = full <= H
        starts = (ptr[:-1].to(i64), split.to(i64))
        lens = (torch.where(light, split.to(i64) - starts[0], 0),
                torch.where(light, ptr[1:].to(i64) - starts[1], 0))
        # "auto": only the slice-padding gate applies (a part whose long rows
        # pad its slices beyond sell_max_pad keeps the CSR-vector split kernels)
        sub = dataclasses.replace(opts, sell_min_nnz=0) if opts.sell == "auto" else opts
        sells, keep = [], []
        for h in range(2):
            ln = lens[h]
            pp = torch.zeros(rows + 1, dtype=i64, device=dev)
            torch.cumsum(ln, 0, out=pp[1:])
            nz = int(pp[-1].item())
            rid = torch.repeat_interleave(torch.arange(rows, device=dev), ln)
            idx = starts[h][rid] + (torch.arange(nz, device=dev) - pp[:-1][rid])
            pcol = col[idx].contiguous()
            pval = val[idx].contiguous()
            p32 = pp.to(torch.int32)
            built = self._build_sell(torch, dev, f"{key}.part{h}", rows, max(nz, 1), p32, pcol, pval, H, sub)
            if built is None:
                return None
            sells.append(built[0])
            keep.append((p32, built[1]))
        return sells, keep

    def _build_psr(self, torch, dev, key, rows, cols, nnz, ptr, col, val, H, opts):
        """Plan + build the PSR layout of one operator on the device (or None)."""
        if opts.psr == "off" or (opts.psr == "auto" and rows < opts.psr_min_rows):
            return None
        if not N.experimental():
            if opts.psr == "auto":
                return None
            raise N.NativeError("psr='on' needs the experiment build of libpdhg_b200 (PSR was measured "
                                "slower; python -m paper_2603_03150_b200.build --experimental and "
                                "PDHG_B200_LIB=tools/_libs/libpdhg_b200_exp.so)")
        lib = self.lib
        sptr = self.stream.cuda_stream
        tb = lib.pdhg_psr_tmp_bytes(rows, cols, nnz)
        tmp = torch.empty(max(tb, 1), dtype=torch.uint8, device=dev)
        R, W, nblk, ngroups, ntiles = (C.c_int32() for _ in range(5))
        staged, nent = C.c_int64(), C.c_int64()
        N.check(lib.pdhg_psr_plan(rows, cols, nnz, ptr.data_ptr(), col.data_ptr(), H,
                                  int(opts.psr_min_staged), tmp.data_ptr(), tb, sptr,
                                  C.byref(R), C.byref(W), C.byref(nblk), C.byref(ngroups),
                                  C.byref(ntiles), C.byref(staged), C.byref(nent)))
        frac = staged.value / max(1, nnz)
        self.psr_info[key] = {"R": R.value, "W": W.value, "nblk": nblk.value, "ntiles": ntiles.value,
                              "ngroups": ngroups.value, "staged_fraction": frac, "nent": nent.value}
        if opts.psr == "auto" and frac < opts.psr_min_fraction:
            return None
        i32 = torch.int32
        nt = max(1, ntiles.value)
        bufs = {
            "blk_tile_ptr": torch.empty(nblk.value + 1, dtype=i32, device=dev),
            "tile_bin": torch.empty(nt, dtype=i32, device=dev),
            "gstart": torch.empty(nt * (ngroups.value + 1), dtype=i32, device=dev),
            "rcnt": torch.empty(nt * ngroups.value * 32, dtype=torch.int16, device=dev),
            "val": torch.empty(max(1, nnz), dtype=torch.float64, device=dev),
            "col16": torch.empty(max(1, nnz), dtype=torch.int16, device=dev),
            "col": torch.empty(max(1, nnz), dtype=i32, device=dev),
            "heavy": torch.empty(rows, dtype=torch.uint8, device=dev),
        }
        names = ("blk_tile_ptr", "tile_bin", "gstart", "rcnt", "val", "col16", "col", "heavy")
        N.check(lib.pdhg_psr_build(rows, cols, nnz, ptr.data_ptr(), col.data_ptr(), val.data_ptr(), H,
                                   tmp.data_ptr(), tb, sptr, *(bufs[k].data_ptr() for k in names)))
        d = N.Psr()
        d.rows, d.cols, d.R, d.W = rows, cols, R.value, W.value
        d.nblk, d.ntiles, d.ngroups, d.nent = nblk.value, ntiles.value, ngroups.value, nent.value
        for k in names:
            setattr(d, k, bufs[k].data_ptr())
        self.psr_info[key]["used"] = True
        return (d, bufs)

    # --- thin wrappers over the C ABI -------------------------------------
    def opnorm(self, v0: np.ndarray, tol: float = 1e-4, max_iters: int = 100) -> float:
        v0 = np.ascontiguousarray(v0, dtype=np.float64)
        lam, its = C.c_double(), C.c_int32()
        if self.col_perm is None:
            N.check(self.lib.pdhg_opnorm(self.ctx, v0.ctypes.data, tol, max_iters,
                                         C.byref(lam), C.byref(its)))
        else:   # renumbered columns: the start vector permuted on the device
            torch = _torch()
            with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
                vd = hostio.h2d(v0, np.float64, self.device).index_select(0, self.col_perm)
                N.check(self.lib.pdhg_opnorm(self.ctx, vd.data_ptr(), tol, max_iters,
                                             C.byref(lam), C.byref(its)))
        self.opnorm_iterations = int(its.value)
        return float(lam.value)

    def reset(self):
        N.check(self.lib.pdhg_reset(self.ctx))

    def run_period(self, iters: int, iter0: int, tau_w: float, sigma_w: float, w0: float) -> int:
        f = C.c_int64()
        N.check(self.lib.pdhg_run_period(self.ctx, int(iters), int(iter0), float(tau_w),
                                         float(sigma_w), float(w0), C.byref(f)))
        return int(f.value)

    def run_period_check(self, iters: int, iter0: int, tau_w: float, sigma_w: float, w0: float,
                         *specs: int):
        """run_period + check(*specs) with one synchronisation -> (fail_iter, [scalars...])."""
        f = C.c_int64()
        arr = (C.c_int32 * max(1, len(specs)))(*specs)
        N.check(self.lib.pdhg_run_period_check(self.ctx, int(iters), int(iter0), float(tau_w),
                                               float(sigma_w), float(w0), len(specs), arr,
                                               C.byref(f), self._scal))
        flat = np.frombuffer(self._scal, dtype=np.float64, count=len(specs) * N.NQ).copy()
        return int(f.value), [flat[k * N.NQ:(k + 1) * N.NQ] for k in range(len(specs))]

    def use_check_dot(self, slot: int) -> None:
        """The next period's first primal step takes A'y of point `slot` of the
        last two-point check (0 = first spec, 1 = second) -- see
        pdhg_use_check_dot in include/pdhg_b200.h."""
        N.check(self.lib.pdhg_use_check_dot(self.ctx, int(slot)))

    def check(self, *specs: int) -> list[np.ndarray]:
        arr = (C.c_int32 * len(specs))(*specs)
        N.check(self.lib.pdhg_check(self.ctx, len(specs), arr, self._scal))
        flat = np.frombuffer(self._scal, dtype=np.float64, count=len(specs) * N.NQ).copy()
        return [flat[k * N.NQ:(k + 1) * N.NQ] for k in range(len(specs))]

    def restart(self, which: int):
        N.check(self.lib.pdhg_restart(self.ctx, which))

    def save_best(self, which: int, flags: int):
        N.check(self.lib.pdhg_save_best(self.ctx, which, flags))

    def fetch(self, spec: int, want_z: bool = True):
        """Host copies of a point (full padded lengths): z computed on the device,
        downloads through the pinned ring (hostio)."""
        torch = _torch()
        px, py, pz = C.c_void_p(), C.c_void_p(), C.c_void_p()
        N.check(self.lib.pdhg_point_device(self.ctx, spec, C.byref(px), C.byref(py), C.byref(pz)))
        base = self.ws.data_ptr()
        view = lambda ptr, k: self.ws[ptr - base:ptr - base + 8 * k].view(torch.float64)
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            xv = view(px.value, self.n_full)
            if self.col_perm is not None:     # renumbered variables -> the caller's order
                xv = xv.index_select(0, self.col_inv)
            x = hostio.d2h(xv)
            yv = view(py.value, self.m_full)
            if self.row_perm is not None:     # renumbered constraints -> the caller's order
                yv = yv.index_select(0, self.row_inv)
            y = hostio.d2h(yv)
            z = None
            if want_z:
                zv = view(pz.value, self.n_full)
                if self.col_perm is not None:
                    zv = zv.index_select(0, self.col_inv)
                z = hostio.d2h(zv)
        return x, y, z

    def _to_cols(self, v: np.ndarray) -> np.ndarray:
        """An x-space host vector in the context's (renumbered) column order."""
        if self.col_perm is None:
            return v
        if self._col_perm_host is None:
            self._col_perm_host = self.col_perm.cpu().numpy()
        return v[self._col_perm_host]

    def spmv(self, v: np.ndarray, transpose: bool = False) -> np.ndarray:
        """A @ v or A' @ v through the device SpMV (the 1e-12 parity gate)."""
        torch = _torch()
        v = np.ascontiguousarray(v, dtype=np.float64)
        if transpose and self.row_perm is not None:
            if self._row_perm_host is None:
                self._row_perm_host = self.row_perm.cpu().numpy()
            v = np.ascontiguousarray(v[self._row_perm_host])
        if not transpose:
            v = np.ascontiguousarray(self._to_cols(v))
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            vin = torch.from_numpy(v).to(self.device)
            out = torch.empty(self.n if transpose else self.m, dtype=torch.float64, device=self.device)
            N.check(self.lib.pdhg_spmv(self.ctx, 1 if transpose else 0, vin.data_ptr(), out.data_ptr()))
            if not transpose and self.row_perm is not None:
                out = out.index_select(0, self.row_inv)
            if transpose and self.col_perm is not None:
                out = out.index_select(0, self.col_inv)
            self.stream.synchronize()
            return out.cpu().numpy()

    # --- sharded-execution building blocks (sharded.py) ---------------------
    def vec(self, name: str):
        """torch float64 view (full padded length) of one of the context's vectors."""
        ptr = self.lib.pdhg_vector(self.ctx, N.VEC[name])
        if not ptr:
            N.check(-1)
        off = ptr - self.ws.data_ptr()
        count = 64 if name == "scalars" else (self.n_full if name in
                                              ("x", "xe", "xbar", "xbest", "zbest", "tn1", "tn2")
                                              else self.m_full)
        return self.ws[off:off + 8 * count].view(self._torch.float64)

    @property
    def _torch(self):
        import torch

        return torch

    def vec_ptr(self, name: str) -> int:
        return self.lib.pdhg_vector(self.ctx, N.VEC[name])

    def set_peers(self, which: int, ptrs):
        """Fused all-gather targets (pdhg_set_peers): which 0 = xe (primal step),
        1 = y (dual step), 2 = the peers' fail words; ptrs = int64 device tensor of
        peer bases (kept alive)."""
        self._peers = getattr(self, "_peers", {})
        self._peers[which] = ptrs
        n = 0 if ptrs is None else int(ptrs.numel())
        N.check(self.lib.pdhg_set_peers(self.ctx, int(which), ptrs.data_ptr() if n else None, n))

    def connect_fail(self, others):
        """Shards on this device: record a non-finite iterate in their fail words too."""
        ptrs = [o.vec_ptr("failword") for o in others]
        self.set_peers(2, self._torch.tensor(ptrs, dtype=self._torch.int64, device=self.device))

    def set_step(self, iter0: int, tau_w: float, sigma_w: float, w0: float):
        N.check(self.lib.pdhg_set_step(self.ctx, int(iter0), float(tau_w), float(sigma_w), float(w0)))

    def half_step(self, primal: bool, j: int):
        N.check(self.lib.pdhg_half_step(self.ctx, 1 if primal else 0, int(j)))

    def half_step_pass(self, primal: bool, j: int, pass_: int):
        """Pass 0 (local-slot entries) or pass 1 (the rest + epilogue) of a split
        half step; an unsplit operator runs whole at pass 0."""
        N.check(self.lib.pdhg_half_step_pass(self.ctx, 1 if primal else 0, int(j), int(pass_)))

    def fail_iter(self) -> int:
        f = C.c_int64()
        N.check(self.lib.pdhg_fail_iter(self.ctx, C.byref(f)))
        return int(f.value)

    def check_device(self, *specs: int):
        arr = (C.c_int32 * len(specs))(*specs)
        N.check(self.lib.pdhg_check_device(self.ctx, len(specs), arr))
        return self.vec("scalars")[:len(specs) * N.NQ]

    def reduced_costs(self, spec: int, out_name: str):
        N.check(self.lib.pdhg_reduced_costs(self.ctx, spec, self.vec_ptr(out_name) + 8 * self.x_off))

    def spmv_named(self, transpose: bool, in_name: str, out_name: str):
        """out[local slice] = (A or A') @ in (full vector)."""
        off = self.x_off if transpose else self.y_off
        N.check(self.lib.pdhg_spmv(self.ctx, 1 if transpose else 0, self.vec_ptr(in_name),
                                   self.vec_ptr(out_name) + 8 * off))

    def sumsq_named(self, name: str):
        """sum of squares of this shard's x-space slice of `name` -> scalars[0] (device)."""
        N.check(self.lib.pdhg_sumsq(self.ctx, self.vec_ptr(name) + 8 * self.x_off, self.n,
                                    self.vec_ptr("scalars")))
        return self.vec("scalars")[:1]

    def div_named(self, src: str, dst: str, s: float):
        N.check(self.lib.pdhg_div(self.ctx, self.vec_ptr(src) + 8 * self.x_off,
                                  self.vec_ptr(dst) + 8 * self.x_off, self.n, float(s)))

    def time_kernel(self, which: int, reps: int, tau_w: float = 0.0, sigma_w: float = 0.0) -> float:
        ms = C.c_double()
        N.check(self.lib.pdhg_time_kernel(self.ctx, which, reps, tau_w, sigma_w, C.byref(ms)))
        return float(ms.value)


# ----------------------------------------------------------------- layout cache

_cache_lock = threading.Lock()
_cache: dict[int, tuple] = {}
_CACHE_MAX = 4


def _fingerprint(p):
    A = p.A
    data = A.data
    step = max(1, data.size // 65536)
    return (A.shape, int(A.nnz), data.ctypes.data, A.indices.ctypes.data, A.indptr.ctypes.data,
            float(np.sum(data[::step])) if data.size else 0.0)


def device_lp(p, opts: GpuOptions) -> DeviceLp:
    """The cached device layout of StandardLp ``p`` (built on first use).

    Cache entries die with ``p`` (weakref) and are rebuilt when A's storage,
    b or c change.  A GPU-side analogue of StandardLp.A_csc (lp_core.py:133-138).
    """
    if not opts.cache_layout:
        return DeviceLp(p.A, p.b, p.c, opts)
    key = id(p)
    fp = _fingerprint(p)
    b = np.asarray(p.b, dtype=float)
    c = np.asarray(p.c, dtype=float)
    with _cache_lock:
        ent = _cache.get(key)
        if ent is not None:
            ref, lay, efp, eb, ec, eopts = ent
            if (ref() is p and efp == fp and eopts == opts and np.array_equal(eb, b)
                    and np.array_equal(ec, c)):
                return lay
            _cache.pop(key, None)
    lay = DeviceLp(p.A, b, c, opts)
    with _cache_lock:
        while len(_cache) >= _CACHE_MAX:
            _cache.pop(next(iter(_cache)))
        try:
            ref = weakref.ref(p, lambda _r, k=key: _cache.pop(k, None))
        except TypeError:  # not weak-referenceable: do not cache
            return lay
        _cache[key] = (ref, lay, fp, b.copy(), c.copy(), GpuOptions(**vars(opts)))
    return lay


def _cache_register(p, lay: DeviceLp, opts: GpuOptions) -> None:
    """Make `lay` the cached device layout of model `p` (used by the device
    Ruiz pass, whose output matrix already lives on the device)."""
    key = id(p)
    try:
        ref = weakref.ref(p, lambda _r, k=key: _cache.pop(k, None))
    except TypeError:
        return
    with _cache_lock:
        while len(_cache) >= _CACHE_MAX:
            _cache.pop(next(iter(_cache)))
        _cache[key] = (ref, lay, _fingerprint(p), np.asarray(p.b, dtype=float).copy(),
                       np.asarray(p.c, dtype=float).copy(), GpuOptions(**vars(opts)))


def clear_cache() -> None:
    with _cache_lock:
        _cache.clear()


# ----------------------------------------------------------------- scores


@dataclass
class _Score:
    """Scalars of one scored point (what _score + residuals give, pdhg.py:154-159)."""

    rp_norm: float
    rd_norm: float
    primal_obj: float
    dual_obj: float
    comp: float
    primal_inf: float
    dual_inf: float
    extra: dict = field(default_factory=dict)


def _score(q: np.ndarray) -> _Score:
    return _Score(
        rp_norm=math.sqrt(q[N.Q_RP2]),   # np.linalg.norm = sqrt(x.x) (lp_core.py:458)
        rd_norm=math.sqrt(q[N.Q_RD2]),
        primal_obj=float(q[N.Q_CX]),     # lp_core.py:441
        dual_obj=float(q[N.Q_BY]),       # lp_core.py:442
        comp=float(q[N.Q_XZ]),           # lp_core.py:443
        primal_inf=float(q[N.Q_RPMAX]),  # lp_core.py:476
        dual_inf=float(q[N.Q_RDMAX]),    # lp_core.py:477
    )


def _summary(T, s: _Score):
    """violation_summary (lp_core.py:468-485) from device scalars."""
    rel_gap = s.comp / (1.0 + abs(s.primal_obj))
    return T.ViolationSummary(
        primal_inf=s.primal_inf, dual_inf=s.dual_inf, rel_gap=rel_gap,
        max_violation=max(s.primal_inf, s.dual_inf, rel_gap), comp_negative=s.comp < 0,
    )


def _termination(T, s: _Score, eps_rel: float, norm_b: float, norm_c: float):
    """check_relative_termination (lp_core.py:447-465) from device scalars."""
    if eps_rel <= 0:
        raise ValueError("eps_rel must be positive")
    p_lhs, d_lhs = s.rp_norm, s.rd_norm
    p_rhs = eps_rel * (1.0 + norm_b)
    d_rhs = eps_rel * (1.0 + norm_c)
    gap_lhs = abs(s.primal_obj - s.dual_obj)
    gap_rhs = eps_rel * (1.0 + abs(s.primal_obj) + abs(s.dual_obj))
    ok = p_lhs <= p_rhs and d_lhs <= d_rhs and gap_lhs <= gap_rhs
    return T.TerminationCheck(ok, p_lhs, p_rhs, d_lhs, d_rhs, gap_lhs, gap_rhs)


# ----------------------------------------------------------------- run_pdhg


def run_pdhg(p, params=None, seed: int = 0, *, gpu: GpuOptions | None = None):
    """Iterate to the requested relative tolerance, restarting adaptively.

    Same contract as hybridlp.pdhg.run_pdhg (pdhg.py:162-258): returns
    (KktPoint, SolveStats); solver outcomes are returned in stats.status,
    never raised; raises InvalidModelError for an empty model or matrix and
    ZeroDivisionError when A holds only explicit zeros (pdhg.py:119).
    """
    T = resolve()
    opts = gpu or GpuOptions()
    if params is None:
        params = T.PdhgParams()
    m, n = p.A.shape
    if m == 0 or n == 0:                                       # pdhg.py:175-176
        raise T.InvalidModelError("pdhg requires a nonempty model")
    t0 = time.monotonic()                                      # pdhg.py:177
    if p.A.nnz == 0:                                           # pdhg.py:87-88
        raise T.InvalidModelError("cannot estimate the norm of an empty matrix")
    v0 = hostio.submit(_start_vector, n, seed) if opts.opnorm is None else None
    dev = device_lp(p, opts)
    t_layout = time.monotonic() - t0
    with dev.lock:
        pt, st = _run(T, dev, p, params, seed, opts, t0, v0)
    if hasattr(st, "timings"):
        st.timings["layout_s"] = t_layout      # device_lp: upload + layout build
        st.timings.update({k: v for k, v in getattr(dev, "timings", {}).items()
                           if k in ("upload_s", "layout_detail")})
    return pt, st


def run_on_device(dev, p, params=None, seed: int = 0, *, gpu: GpuOptions | None = None):
    """run_pdhg's control flow over an already-built device (DeviceLp or
    sharded.ShardedDevice).  The clock starts here, after the layout build."""
    T = resolve()
    if params is None:
        params = T.PdhgParams()
    t0 = time.monotonic()
    return _run(T, dev, p, params, seed, gpu or GpuOptions(), t0)


def _start_vector(n: int, seed: int) -> np.ndarray:
    """The power iteration's start vector, exactly the reference's
    (pdhg.py:89-91: default_rng(seed).standard_normal(n), normalised)."""
    v = np.random.default_rng(seed).standard_normal(n)
    v /= np.linalg.norm(v)
    return v


def _run(T, dev: DeviceLp, p, params, seed, opts, t0, v0_future=None):
    S = T.SolveStatus
    b = np.asarray(p.b, dtype=float)
    c = np.asarray(p.c, dtype=float)
    norm_b = float(np.linalg.norm(b)) if b.size else 0.0       # lp_core.py:460
    norm_c = float(np.linalg.norm(c)) if c.size else 0.0       # lp_core.py:461
    eps = params.eps_rel

    tm = {}
    t_op = time.monotonic()
    # initial_state (pdhg.py:117-137)
    if opts.opnorm is not None:
        opnorm = float(opts.opnorm)
    else:
        # generated on a host thread while the model was uploaded (run_pdhg)
        v = v0_future.result() if v0_future is not None else _start_vector(dev.n, seed)
        opnorm = dev.opnorm(v, tol=1e-4, max_iters=100)
    step = 1.0 / (1.05 * opnorm)                               # pdhg.py:119
    tm["opnorm_s"] = time.monotonic() - t_op
    if getattr(dev, "opnorm_iterations", None) is not None and opts.opnorm is None:
        tm["opnorm_iterations"] = dev.opnorm_iterations
    t_it = time.monotonic()
    dev.reset()
    tau = sigma = step
    omega = params.primal_weight_init
    iterations = 0
    restarts = 0
    avg_weight = 0.0

    (q0,) = dev.check(N.PT_CUR)
    zero_sum = _summary(T, _score(q0))
    restart_score = zero_sum.max_violation                     # pdhg.py:122,136
    # best_pt = zero point (pdhg.py:180): a frozen snapshot
    dev.save_best(N.PT_CUR, N.BEST_XY | N.BEST_Z)
    best_summary = zero_sum
    best_live_avg = False   # True: best x,y alias the running average (see module doc)
    status = S.ITERATION_LIMIT
    history = []
    check_every = int(params.check_every)

    while True:
        if iterations >= params.max_kkt_passes:                # pdhg.py:185-187
            status = S.ITERATION_LIMIT
            break
        timed_out = time.monotonic() - t0 > params.time_limit_s   # pdhg.py:188-190
        if hasattr(dev, "agree") and math.isfinite(params.time_limit_s):
            timed_out = dev.agree(timed_out)    # shards stop together (clocks differ per rank)
        if timed_out:
            status = S.TIME_LIMIT
            break
        k = min(check_every - iterations % check_every, int(params.max_kkt_passes) - iterations)
        at_check = (iterations + k) % check_every == 0
        if at_check and hasattr(dev, "run_period_check"):      # one sync for steps + check
            fail, qs = dev.run_period_check(k, iterations, tau / omega, sigma * omega, avg_weight,
                                            N.PT_CUR, N.PT_AVG)
        else:
            fail, qs = dev.run_period(k, iterations, tau / omega, sigma * omega, avg_weight), None
        if fail >= 0:                                          # pdhg.py:194-196
            avg_weight += fail - iterations
            iterations = fail
            status = S.NUMERICAL_FAILURE
            break
        iterations += k
        avg_weight += k
        if iterations % check_every != 0:                      # pdhg.py:198-199
            continue

        q_cur, q_avg = qs if qs is not None else dev.check(N.PT_CUR, N.PT_AVG)  # pdhg.py:201-204
        s_cur, s_avg = _score(q_cur), _score(q_avg)
        cur_sum, avg_sum = _summary(T, s_cur), _summary(T, s_avg)
        cur_term = _termination(T, s_cur, eps, norm_b, norm_c)
        avg_term = _termination(T, s_avg, eps, norm_b, norm_c)
        rec = {
            "iteration": iterations, "omega": omega, "restart": False,
            "cur_max_violation": cur_sum.max_violation, "avg_max_violation": avg_sum.max_violation,
            "cur_termination": cur_term, "avg_termination": avg_term,
        }
        history.append(rec)

        passing = [(which, term, s) for which, term, s in
                   ((N.PT_CUR, cur_term, cur_sum), (N.PT_AVG, avg_term, avg_sum)) if term.ok]
        if passing:                                            # pdhg.py:214-224
            which, term, summ = min(passing, key=lambda t: t[2].max_violation)
            tm["iterate_s"] = time.monotonic() - t_it
            t_f = time.monotonic()
            x, y, z = dev.fetch(which)
            tm["fetch_s"] = time.monotonic() - t_f
            stats = T.SolveStats(
                status=S.OPTIMAL, iterations=iterations, restarts=restarts,
                wall_seconds=time.monotonic() - t0, termination=term,
                max_violation=summ.max_violation, history=history, timings=tm,
            )
            return T.KktPoint(x, y, z), stats

        if avg_sum.max_violation < cur_sum.max_violation:      # pdhg.py:226-229
            cand, cand_sum, cand_s = N.PT_AVG, avg_sum, s_avg
        else:
            cand, cand_sum, cand_s = N.PT_CUR, cur_sum, s_cur

        if cand_sum.max_violation < best_summary.max_violation:  # pdhg.py:231-232
            best_summary = cand_sum
            if cand == N.PT_CUR:
                dev.save_best(N.PT_CUR, N.BEST_XY | N.BEST_Z)
                best_live_avg = False
            else:
                dev.save_best(N.PT_AVG, N.BEST_Z)
                best_live_avg = True

        restarted = False
        if cand_sum.max_violation <= params.restart_beta * restart_score:  # pdhg.py:234-247
            if best_live_avg:  # the average array best_pt aliases is rebound: freeze it
                dev.save_best(N.PT_AVG, N.BEST_XY)
                best_live_avg = False
            dev.restart(cand)
            restarted = True
            avg_weight = 0.0
            rp, rd = cand_s.rp_norm, cand_s.rd_norm
            if rp > 0.0 and rd > 0.0:
                omega = float(np.clip(rp / rd, *_WEIGHT_CLIP))
            restart_score = cand_sum.max_violation
            restarts += 1
            rec["restart"] = True
        if getattr(dev, "check_dot", False):
            # the next iterate's y is the current point's, or the average's after
            # a restart to it: the check already holds its A'y (pdhg_use_check_dot)
            dev.use_check_dot(1 if (restarted and cand == N.PT_AVG) else 0)

    # failure exit (pdhg.py:249-258): best point, re-checked with its own z
    tm["iterate_s"] = time.monotonic() - t_it
    t_f = time.monotonic()
    spec = (N.PT_AVG if best_live_avg else N.PT_BEST) | N.SPEC_BEST_Z
    (q_best,) = dev.check(spec)
    termination = _termination(T, _score(q_best), eps, norm_b, norm_c)
    x, y, z = dev.fetch(spec)
    tm["fetch_s"] = time.monotonic() - t_f
    stats = T.SolveStats(
        status=status, iterations=iterations, restarts=restarts,
        wall_seconds=time.monotonic() - t0, termination=termination,
        max_violation=best_summary.max_violation, history=history, timings=tm,
    )
    return T.KktPoint(x, y, z), stats


def estimate_opnorm(A, seed: int = 0, tol: float = 1e-4, max_iters: int = 100,
                    *, gpu: GpuOptions | None = None) -> float:
    """Device power iteration with the reference's start vector (pdhg.py:80-109)."""
    T = resolve()
    m, n = A.shape
    if m == 0 or n == 0 or A.nnz == 0:
        raise T.InvalidModelError("cannot estimate the norm of an empty matrix")

    class _P:  # minimal StandardLp stand-in
        pass

    q = _P()
    q.A, q.b, q.c = A, np.zeros(m), np.zeros(n)
    dev = DeviceLp(A, q.b, q.c, gpu or GpuOptions())
    return dev.opnorm(_start_vector(n, seed), tol=tol, max_iters=max_iters)
