"""Multi-GPU execution of the PDHG path: row/column sharding with all-gathers.

Design.  For G shards:

* rows of A are cut into G contiguous blocks of ~equal nnz (shard g owns
  y-space rows [r_g, r_{g+1})), and columns of A -- rows of A' -- likewise
  (shard g owns x-space rows [c_g, c_{g+1}));
* every vector is stored at full, *padded* length: slice g of the y-space
  vector is [g*maxR, g*maxR + (r_{g+1}-r_g)) with maxR = max block height,
  so every slice has the same size and an in-place all-gather of equal
  chunks completes the vector; matrix indices are remapped to these slots
  once, on the host (monotone, so CSR column order is kept);
* per iteration: primal half step on A' rows (gathers full y, writes the
  x / xe / avg_x slice) -> all-gather xe -> dual half step on A rows
  (gathers full xe, writes the y / avg_y slice) -> all-gather y;
* at a check every shard scores its own rows; the per-shard partial sums and
  maxima are all-gathered and combined in rank order, so every rank takes
  the identical restart / termination decision (pdhg.py:206-247).

``ShardedDevice`` exposes the same interface engine._run drives for one GPU
(opnorm, reset, run_period, check, restart, save_best, fetch), so the host
control flow is shared verbatim.  A shard backend is a DeviceLp (CUDA
kernels behind the C ABI); a communicator moves slices between shards:

* ``TorchComm``    -- one shard per process, torch.distributed all_gather
                      (NCCL over NVLink on a B200 box; gloo in CPU tests);
* ``LoopbackComm`` -- all G shards in one process on one device (tests the
                      sharded kernels and the rank-order combine on 1 GPU);
                      the all-gather is a set of device-to-device copies;
* fused all-gather (``fused=True``): the step kernels' epilogues store each
  new xe / y value straight into every peer's full vector at the shard's
  slot (``pdhg_set_peers``), so no all-gather runs after a half step.  In
  loopback the peers are the other shards' buffers on the same device
  (stream order is the barrier); with ``comm_kind="torch_peer"`` the
  workspace is torch symmetric memory, the peers are NVLink addresses
  (``buffer_ptrs``) and a symmetric-memory barrier on the stream orders
  each half step after every rank's stores.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _native as N

X_SPACE = ("x", "xe", "xbar", "xbest", "zbest", "tn1", "tn2")
Y_SPACE = ("y", "ybar", "ybest", "tm1")


# ----------------------------------------------------------------- partition


def _cuts(counts_ptr: np.ndarray, G: int) -> np.ndarray:
    """G+1 strictly increasing cut points over rows with ~equal entries
    (ptr = cumulative counts).  Every shard owns at least one row: a row
    holding >= nnz/G entries (a dense linking row) would otherwise give two
    shards the same cut and one of them no rows."""
    total = int(counts_ptr[-1])
    rows = counts_ptr.size - 1
    if rows < G:
        raise ValueError(f"cannot shard {rows} rows over {G} shards")
    cuts = [0]
    for g in range(1, G):
        c = int(np.searchsorted(counts_ptr, g * total / G, side="left"))
        cuts.append(min(max(c, cuts[-1] + 1), rows - (G - g)))
    cuts.append(rows)
    return np.asarray(cuts, dtype=np.int64)


def _local_first(M: sp.csr_matrix, lo: int, hi: int):
    """Reorder each row's entries: columns in [lo, hi) first, then the rest,
    each part keeping its order; returns (matrix, per-row count of the first part)."""
    rows = M.shape[0]
    lens = np.diff(M.indptr)
    rid = np.repeat(np.arange(rows, dtype=np.int64), lens)
    remote = (M.indices < lo) | (M.indices >= hi)
    order = np.argsort(rid * 2 + remote, kind="stable")
    nloc = np.bincount(rid[~remote], minlength=rows).astype(np.int32)
    out = sp.csr_matrix((M.data[order], M.indices[order], M.indptr.copy()), shape=M.shape)
    out.has_sorted_indices = False
    return out, nloc


@dataclass
class ShardBlock:
    """What shard g needs: its A rows, its A' rows, b/c slices and slice offsets."""

    g: int
    A: sp.csr_matrix       # rows [r_g, r_g+1) of A, columns in x-space slots (width n_full)
    At: sp.csr_matrix      # rows [c_g, c_g+1) of A', columns in y-space slots (width m_full)
    b: np.ndarray
    c: np.ndarray
    m_full: int
    n_full: int
    y_off: int
    x_off: int
    # local_first blocks: each row holds its entries in this shard's own slot
    # range first (a_nloc / at_nloc of them), then the others, each part in
    # column order -- the split steps' pass 0 / pass 1
    a_nloc: np.ndarray | None = None
    at_nloc: np.ndarray | None = None


def block_length_order(lens: np.ndarray, rcut: np.ndarray, window: int, first: int = 0) -> np.ndarray:
    """New position -> old row: inside every row block [rcut[g], rcut[g+1]),
    rows by decreasing length within windows of `window` rows (stable) --
    the single-GPU renumbering (engine._length_order) applied per shard, so
    every block keeps its rows and with them its band of local columns; with
    first > 0 the block's rows longer than `first` come first (window by
    window), then the rest."""
    order = np.arange(lens.size, dtype=np.int64)
    for g in range(rcut.size - 1):
        r0, r1 = int(rcut[g]), int(rcut[g + 1])
        if r1 - r0 < 2:
            continue
        ln = lens[r0:r1].astype(np.int64)
        top = int(ln.max()) + 1
        win = np.arange(r1 - r0, dtype=np.int64) // max(1, int(window))
        key = win * (top + 1) + (top - ln)
        if first > 0:
            key = (ln <= first).astype(np.int64) * (int(win[-1]) + 1) * (top + 1) + key
        order[r0:r1] = r0 + np.argsort(key, kind="stable")
    return order


class ShardPlan:
    """Equal-nnz row and column partition of A over G shards, with padded slots.

    ``row_window`` > 0: inside each row block the constraints are renumbered
    by decreasing length in windows of that many rows (block_length_order) --
    the block's slot k holds original row rorder[r_g + k], yslot maps every
    original row to its slot, so the A' blocks (indexed by slot), the
    all-gathers and the result download (y = slots[yslot]) follow without
    further change.  Each row's entries and each A' row's entry order are
    unchanged, so the steps' sums are those of the unrenumbered plan; the
    sliced-ELL slices of A's blocks lose their long-row padding.
    ``first`` > 0: inside each block, the rows / variables longer than
    that come first (window by window), as the single-GPU renumbering does.
    ``col_window`` > 0: the same for the variables inside each column block
    (A' rows; corder / xslot), which also carries the power iteration's start
    vector and the x / z download."""

    def __init__(self, A, G: int, row_window: int = 0, col_window: int = 0, first: int = 0):
        A = sp.csr_matrix(A)
        self.G = int(G)
        self.m, self.n = A.shape
        self.nnz = int(A.nnz)
        self.rcut = _cuts(np.asarray(A.indptr, dtype=np.int64), self.G)
        col_counts = np.bincount(A.indices, minlength=self.n)
        cptr = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(col_counts, out=cptr[1:])
        self.ccut = _cuts(cptr, self.G)
        self.maxR = max(1, int(np.max(np.diff(self.rcut))))
        self.maxC = max(1, int(np.max(np.diff(self.ccut))))
        self.m_full = self.G * self.maxR
        self.n_full = self.G * self.maxC
        rg = np.repeat(np.arange(self.G), np.diff(self.rcut))
        cg = np.repeat(np.arange(self.G), np.diff(self.ccut))
        self.yslot = (rg * self.maxR + np.arange(self.m) - self.rcut[rg]).astype(np.int64)
        self.xslot = (cg * self.maxC + np.arange(self.n) - self.ccut[cg]).astype(np.int64)
        self.row_window = int(row_window)
        self.rorder = None
        if self.row_window > 0:
            self.rorder = block_length_order(np.diff(A.indptr), self.rcut, self.row_window, first)
            slots = self.yslot.copy()
            self.yslot[self.rorder] = slots          # the row at new position p takes p's slot
        self.col_window = int(col_window)
        self.corder = None
        if self.col_window > 0:
            self.corder = block_length_order(col_counts, self.ccut, self.col_window, first)
            slots = self.xslot.copy()
            self.xslot[self.corder] = slots

    def block(self, g: int, A, b, c, local_first: bool = False) -> ShardBlock:
        """Shard g's rows of A and of A' (slot-indexed).  ``local_first``: each
        row's entries in g's own slot range first (for the overlapped
        schedule's split steps), with their counts in a_nloc / at_nloc."""
        A = A if sp.isspmatrix_csr(A) else sp.csr_matrix(A)
        r0, r1 = int(self.rcut[g]), int(self.rcut[g + 1])
        c0, c1 = int(self.ccut[g]), int(self.ccut[g + 1])
        rows = slice(r0, r1) if self.rorder is None else self.rorder[r0:r1]
        Ar = A[rows]
        Ag = sp.csr_matrix((Ar.data, self.xslot[Ar.indices].astype(np.int32), Ar.indptr),
                           shape=(r1 - r0, self.n_full))
        # CSC of A once per plan (column blocks are then contiguous ranges) =
        # CSR of the transpose's row blocks
        if getattr(self, "_csc_of", None) is not A:
            self._csc, self._csc_of = A.tocsc(), A
        Acsc = self._csc
        if self.corder is None:
            s0, s1 = int(Acsc.indptr[c0]), int(Acsc.indptr[c1])
            Atg = sp.csr_matrix((Acsc.data[s0:s1], self.yslot[Acsc.indices[s0:s1]].astype(np.int32),
                                 (Acsc.indptr[c0:c1 + 1] - s0).astype(Acsc.indptr.dtype)),
                                shape=(c1 - c0, self.m_full))
            cols = slice(c0, c1)
        else:   # renumbered variables: the block's columns in corder (each keeps its entry order)
            cols = self.corder[c0:c1]
            sub = Acsc[:, cols]
            Atg = sp.csr_matrix((sub.data, self.yslot[sub.indices].astype(np.int32), sub.indptr),
                                shape=(c1 - c0, self.m_full))
        blk = ShardBlock(g, Ag, Atg, np.asarray(b, float)[rows], np.asarray(c, float)[cols],
                         self.m_full, self.n_full, g * self.maxR, g * self.maxC)
        if local_first:
            blk.A, blk.a_nloc = _local_first(Ag, g * self.maxC, (g + 1) * self.maxC)
            blk.At, blk.at_nloc = _local_first(Atg, g * self.maxR, (g + 1) * self.maxR)
        return blk

    def slice_len(self, space: str) -> int:
        return self.maxC if space == "x" else self.maxR


# ------------------------------------------------------------- communicators


class LoopbackComm:
    """All shards in this process (one device): all-gather = device copies."""

    def __init__(self, plan: ShardPlan, fused: bool = False):
        self.plan = plan
        self.rank, self.world = 0, plan.G
        self.local = list(range(plan.G))
        self.fused = fused

    def connect_peers(self, shards):
        """Fused all-gather: shard g's epilogues also write the other shards' xe / y."""
        import torch

        for g, s in enumerate(shards):
            for which, name in ((0, "xe"), (1, "y")):
                ptrs = [o.vec_ptr(name) for h, o in enumerate(shards) if h != g]
                s.set_peers(which, torch.tensor(ptrs, dtype=torch.int64, device=s.device))

    def connect_fail(self, shards):
        """A non-finite iterate on any shard stops every shard at that iteration
        (as on one GPU): each shard's epilogues also record it in the others'
        fail words."""
        for g, s in enumerate(shards):
            others = [o for h, o in enumerate(shards) if h != g]
            if others:
                s.connect_fail(others)
        self.fail_connected = True

    def barrier(self, shards):
        pass   # one stream: stream order is the barrier

    def allgather(self, shards, name: str):
        L = self.plan.slice_len("x" if name in X_SPACE else "y")
        views = [s.vec(name) for s in shards]
        for g, src in enumerate(views):
            part = src[g * L:(g + 1) * L]
            for h, dst in enumerate(views):
                if h != g:
                    dst[g * L:(g + 1) * L].copy_(part)

    def gather_rows(self, shards, per_shard):
        """per_shard: one device tensor per local shard -> (G, k) numpy, rank order."""
        return np.stack([t.double().cpu().numpy() for t in per_shard])

    def allgather_int(self, value_per_shard):
        return list(value_per_shard)


class TorchComm:
    """One shard per process over torch.distributed (NCCL on GPUs, gloo in tests)."""

    def __init__(self, plan: ShardPlan, group=None, fused: bool = False):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.plan = plan
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world != plan.G:
            raise ValueError("world size must equal the number of shards")
        self.local = [self.rank]
        self.fused = fused
        self.symm = None

    def symmetric_workspace(self, nbytes: int, device):
        """Workspace allocator for the fused mode: torch symmetric memory (identical
        size on every rank -- the padded layout makes it so)."""
        import torch.distributed._symmetric_memory as symm_mem
        import torch

        return symm_mem.empty(nbytes, dtype=torch.uint8, device=device)

    def connect_peers(self, shards):
        """Peer vector bases over NVLink: the symmetric workspace's buffer_ptrs plus
        the (rank-independent) offsets of xe / y inside it."""
        import torch
        import torch.distributed._symmetric_memory as symm_mem

        (s,) = shards
        self.symm = symm_mem.rendezvous(s.ws, self.group or self.dist.group.WORLD)
        base = s.ws.data_ptr()
        for which, name in ((0, "xe"), (1, "y"), (2, "failword")):
            off = s.vec_ptr(name) - base
            ptrs = [int(self.symm.buffer_ptrs[r]) + off for r in range(self.world) if r != self.rank]
            if which < 2 or ptrs:
                s.set_peers(which, torch.tensor(ptrs, dtype=torch.int64, device=s.device))

    def connect_fail(self, shards):
        pass   # done in connect_peers (the fail words live in the symmetric workspace)

    def barrier(self, shards):
        """Stream-ordered cross-GPU barrier: the next half step starts after every
        rank's epilogue stores.  torch's symmetric-memory barrier is a kernel on
        the current stream: each rank sets its slot in every peer's signal pad
        and waits for every peer's slot in its own (release / acquire, the
        waiter resets the slot), so it is captured into the period graph."""
        self.symm.barrier(channel=0)

    def allgather(self, shards, name: str):
        (s,) = shards
        L = self.plan.slice_len("x" if name in X_SPACE else "y")
        full = s.vec(name)[:L * self.world]
        mine = full[self.rank * L:(self.rank + 1) * L].clone()
        self.dist.all_gather_into_tensor(full, mine, group=self.group)

    def gather_rows(self, shards, per_shard):
        import torch

        (t,) = per_shard
        out = torch.empty((self.world, t.numel()), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out.view(-1), t.contiguous(), group=self.group)
        return out.double().cpu().numpy()

    def allgather_int(self, value_per_shard):
        import torch

        (v,) = value_per_shard
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([int(v)], dtype=torch.int64, device=dev)
        out = torch.empty(self.world, dtype=torch.int64, device=dev)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return [int(u) for u in out.cpu()]


# --------------------------------------------------------------- the device


def _combine(rows: np.ndarray, npts: int) -> list[np.ndarray]:
    """Rank-order combine of per-shard check partials: sums left to right,
    maxima with NaN propagation (np.max semantics)."""
    out = []
    for p in range(npts):
        blk = rows[:, p * N.NQ:(p + 1) * N.NQ]
        q = np.zeros(N.NQ)
        for k in range(N.NQ):
            if k in (N.Q_RPMAX, N.Q_RDMAX):
                v = blk[0, k]
                for r in range(1, blk.shape[0]):
                    w = blk[r, k]
                    v = w if (w != w or w > v) and v == v else v
                q[k] = v
            else:
                acc = 0.0
                for r in range(blk.shape[0]):
                    acc = acc + float(blk[r, k])
                q[k] = acc
        out.append(q)
    return out


class ShardedDevice:
    """G shards behind engine._run's device interface (see module doc)."""

    def __init__(self, plan: ShardPlan, shards, comm, graph: bool = True, overlap: str = "off"):
        """overlap: "on" -- split half steps (local-first blocks) with each
        all-gather on a side stream, overlapping pass 0;
        "serial" -- the same split kernels and all-gathers on one stream (the
        bitwise reference for "on"); "off" -- unsplit half steps."""
        if overlap not in ("off", "on", "serial"):
            raise ValueError(f"overlap must be 'off', 'on' or 'serial', not {overlap!r}")
        self.plan = plan
        self.shards = list(shards)   # local shard backends, in comm.local order
        self.comm = comm
        self.overlap = overlap
        if overlap == "on" and (getattr(comm, "fused", False)
                                or any(getattr(sh, "stream", None) is None for sh in self.shards)):
            self.overlap = "serial"   # fused stores / CPU doubles: no side stream to overlap on
        self._comm_stream = None
        self.m, self.n = plan.m, plan.n
        # a period (kernels + all-gathers or peer stores + barriers) is captured
        # once per length and replayed, like the single-GPU engine's graphs
        # the fused peer-store mode is captured too: its barrier is a device-side
        # kernel on the stream (symmetric-memory signal pads, each slot set by
        # the peer and reset by its waiter -- replay-safe), not a host wait
        self.graph = graph and all(getattr(sh, "stream", None) is not None for sh in self.shards)
        self._graphs = {}
        self._seen = set()

    def _on_stream(self):
        """torch work (copies, collectives) must queue behind the kernels on
        the shards' stream (loopback shards share one stream)."""
        import contextlib

        st = getattr(self.shards[0], "stream", None)
        if st is None:
            return contextlib.nullcontext()
        import torch

        return torch.cuda.stream(st)

    def _ag(self, *names):
        with self._on_stream():
            for nm in names:
                self.comm.allgather(self.shards, nm)

    # -- power iteration (pdhg.py:80-109), host-driven across shards
    def opnorm(self, v0: np.ndarray, tol: float = 1e-4, max_iters: int = 100) -> float:
        full = np.zeros(self.plan.n_full)
        full[self.plan.xslot] = v0
        with self._on_stream():
            for s in self.shards:
                s.vec("tn1").copy_(_to_like(full, s.vec("tn1")))
        lam = 0.0
        for _ in range(max_iters):
            norm_w = self._aat_norm()
            if norm_w == 0.0:
                break
            new_lam = math.sqrt(norm_w)
            for s in self.shards:
                s.div_named("tn2", "tn1", norm_w)
            self._ag("tn1")
            if lam > 0 and abs(new_lam - lam) <= tol * new_lam:
                lam = new_lam
                break
            lam = new_lam
        norm_w = self._aat_norm()
        if norm_w > 0:
            lam = max(lam, float(math.sqrt(norm_w)))
        return float(lam)

    def _aat_norm(self) -> float:
        for s in self.shards:
            s.spmv_named(False, "tn1", "tm1")
        self._ag("tm1")
        for s in self.shards:
            s.spmv_named(True, "tm1", "tn2")
        with self._on_stream():
            parts = self.comm.gather_rows(self.shards, [s.sumsq_named("tn2") for s in self.shards])
        ss = 0.0
        for r in range(parts.shape[0]):
            ss = ss + float(parts[r, 0])
        return math.sqrt(ss)

    def reset(self):
        for s in self.shards:
            s.reset()

    def _shared_fail(self) -> bool:
        """Do the shards see each other's fail words during a period?  (fused
        peer stores carry them over NVLink; loopback shards after connect_fail)"""
        return bool(getattr(self.comm, "fused", False) or getattr(self.comm, "fail_connected", False)
                    or self.plan.G == 1)

    def _snapshot(self):
        """Each shard's own slices of the iterate vectors at the period start."""
        snap = []
        with self._on_stream():
            for s in self.shards:
                xs, ys = slice(s.x_off, s.x_off + s.n), slice(s.y_off, s.y_off + s.m)
                snap.append({nm: s.vec(nm)[xs if nm in X_SPACE else ys].clone()
                             for nm in ("x", "xe", "xbar", "y", "ybar")})
        return snap

    def _restore(self, snap):
        with self._on_stream():
            for s, d in zip(self.shards, snap):
                xs, ys = slice(s.x_off, s.x_off + s.n), slice(s.y_off, s.y_off + s.m)
                for nm, t in d.items():
                    s.vec(nm)[xs if nm in X_SPACE else ys].copy_(t)
        self._ag("y")           # the full y every shard gathers in the first primal step

    def run_period(self, iters: int, iter0: int, tau_w: float, sigma_w: float, w0: float) -> int:
        # Without shared fail words (the NCCL all-gather mode) a shard does not
        # see another's non-finite iterate until the period ends, and keeps
        # stepping.  Then the period is replayed from a snapshot of its start up
        # to the failing iteration exactly, so every shard stops there as on one
        # GPU (pdhg.py:194-196) -- deterministic kernels make the replay the
        # same arithmetic.  The snapshot is five slice copies per period.
        snap = self._snapshot() if iters > 0 and not self._shared_fail() else None
        fail = self._run_period(iters, iter0, tau_w, sigma_w, w0)
        if snap is not None and fail >= 0:
            self._restore(snap)
            for s in self.shards:
                s.set_step(iter0, tau_w, sigma_w, w0)
            self._period_body(fail - iter0)
            with self._on_stream():
                fails = self.comm.allgather_int([s.fail_iter() for s in self.shards])
            bad = [f for f in fails if f >= 0]
            fail = min(bad) if bad else fail
        return fail

    def _run_period(self, iters: int, iter0: int, tau_w: float, sigma_w: float, w0: float) -> int:
        for s in self.shards:
            s.set_step(iter0, tau_w, sigma_w, w0)
        if self.graph and iters > 0 and iters in self._seen:
            g = self._graphs.get(iters)
            if g is None:
                g = self._capture(iters)
            with self._on_stream():
                g.replay()
        else:
            self._period_body(iters)
            self._seen.add(iters)   # first run eager (lazy NCCL / allocator init), then capture
        with self._on_stream():
            fails = self.comm.allgather_int([s.fail_iter() for s in self.shards])
        bad = [f for f in fails if f >= 0]
        return min(bad) if bad else -1

    def _capture(self, iters: int):
        import torch

        st = self.shards[0].stream
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            self._period_body(iters)
        self._graphs[iters] = g
        return g

    def _side_stream(self):
        import torch

        if self._comm_stream is None:
            self._comm_stream = torch.cuda.Stream(self.shards[0].stream.device)
        return self._comm_stream

    def _period_split(self, iters: int):
        """Split half steps.  overlap="on": per half step, pass 0 (the shard's
        local-slot entries) runs while the other shards' slices of the vector it
        just produced are all-gathered on a side stream; pass 1 (remote entries
        + epilogue) waits for that all-gather.  "serial": the same on one stream."""
        import contextlib

        import torch

        side = self.overlap == "on"
        main = self.shards[0].stream
        comm = self._side_stream() if side else None
        pending = None                  # event: last all-gather (of y) done on the side stream

        def gather(name):
            if not side:
                self._ag(name)
                return None
            ev = torch.cuda.Event()
            ev.record(main)
            comm.wait_event(ev)
            with torch.cuda.stream(comm):
                self.comm.allgather(self.shards, name)
            done = torch.cuda.Event()
            done.record(comm)
            return done

        with torch.cuda.stream(main) if main is not None else contextlib.nullcontext():
            for j in range(iters):
                for sh in self.shards:
                    sh.half_step_pass(True, j, 0)
                if pending is not None:
                    main.wait_event(pending)
                for sh in self.shards:
                    sh.half_step_pass(True, j, 1)
                done_x = gather("xe")
                for sh in self.shards:
                    sh.half_step_pass(False, j, 0)
                if done_x is not None:
                    main.wait_event(done_x)
                for sh in self.shards:
                    sh.half_step_pass(False, j, 1)
                pending = gather("y")
            if pending is not None:
                main.wait_event(pending)

    def _period_body(self, iters: int):
        """The kernels and all-gathers of one period, queued on the shards' stream."""
        if self.overlap in ("on", "serial") and iters > 0:
            return self._period_split(iters)
        fused = getattr(self.comm, "fused", False)
        if fused and iters > 0:         # every rank has reset its fail word (set_step)
            with self._on_stream():
                self.comm.barrier(self.shards)
        for j in range(iters):
            for s in self.shards:
                s.half_step(True, j)
            if fused:                   # xe slices already pushed by the epilogues
                with self._on_stream():
                    self.comm.barrier(self.shards)
            else:
                self._ag("xe")
            for s in self.shards:
                s.half_step(False, j)
            if fused:
                with self._on_stream():
                    self.comm.barrier(self.shards)
            else:
                self._ag("y")

    def agree(self, flag: bool) -> bool:
        """True on every rank if it is true on any (the time-limit exit): each
        rank reads its own clock, the decision must be collective."""
        with self._on_stream():
            flags = self.comm.allgather_int([int(bool(flag))] * len(self.shards))
        return any(flags)

    def _complete(self, spec: int):
        which = spec & 3
        xs = {N.PT_CUR: "x", N.PT_AVG: "xbar", N.PT_BEST: "xbest"}[which]
        ys = {N.PT_CUR: "y", N.PT_AVG: "ybar", N.PT_BEST: "ybest"}[which]
        self._ag(xs, ys)

    def check(self, *specs: int):
        for sp_ in specs:
            self._complete(sp_)
        with self._on_stream():
            rows = self.comm.gather_rows(self.shards, [s.check_device(*specs) for s in self.shards])
        return _combine(rows, len(specs))

    def restart(self, which: int):
        self._complete(which)
        for s in self.shards:
            s.restart(which)

    def save_best(self, which: int, flags: int):
        self._complete(which)
        for s in self.shards:
            s.save_best(which, flags)

    def fetch(self, spec: int, want_z: bool = True):
        self._complete(spec)
        if want_z:
            if spec & N.SPEC_BEST_Z:
                self._ag("zbest")
                zname = "zbest"
            else:
                for s in self.shards:
                    s.reduced_costs(spec, "tn1")
                self._ag("tn1")
                zname = "tn1"
        which = spec & 3
        xs = {N.PT_CUR: "x", N.PT_AVG: "xbar", N.PT_BEST: "xbest"}[which]
        ys = {N.PT_CUR: "y", N.PT_AVG: "ybar", N.PT_BEST: "ybest"}[which]
        s0 = self.shards[0]
        with self._on_stream():
            x = _np(s0.vec(xs))[self.plan.xslot]
            y = _np(s0.vec(ys))[self.plan.yslot]
            z = _np(s0.vec(zname))[self.plan.xslot] if want_z else None
        return x, y, z


def _np(t) -> np.ndarray:
    return t.detach().cpu().numpy().copy()


def _to_like(a: np.ndarray, like):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(like.device)


# ----------------------------------------------------------- entry points


def shard_windows(opts, A) -> tuple[int, int, int]:
    """ShardPlan's (row_window, col_window, first) for GpuOptions.row_order /
    col_order: "length" -> the renumbering window, "natural" -> 0, "auto" ->
    the window when A's rows average >= sell_max_mean entries (long,
    lognormal-tailed rows whose sliced-ELL slices the renumbering un-pads;
    config 4), else 0 -- the variables follow the constraints' choice, as on
    one GPU."""
    if opts is None:
        from .engine import GpuOptions

        opts = GpuOptions()
    auto = A.shape[0] > 0 and A.nnz / A.shape[0] >= opts.sell_max_mean
    win = int(opts.row_order_window)
    rw = win if opts.row_order == "length" or (opts.row_order == "auto" and auto) else 0
    cw = win if opts.col_order == "length" or (opts.col_order == "auto" and rw > 0) else 0
    return rw, cw, int(opts.row_order_first)


def build_sharded(p, G: int, comm_kind: str = "loopback", opts=None, group=None, overlap: str = "auto"):
    """ShardedDevice for StandardLp ``p`` over G shards of CUDA contexts.

    comm_kind="loopback": all G shards on the current device (one process);
    comm_kind="torch": this process's shard (rank) of a torch.distributed job.
    overlap: "on" / "serial" / "off" (ShardedDevice); "auto" = "on" for the
    NCCL all-gather mode ("torch"), "off" otherwise.
    """
    import torch

    from .engine import DeviceLp, GpuOptions

    opts = opts or GpuOptions()
    if overlap == "auto":
        overlap = "on" if comm_kind == "torch" else "off"
    split = overlap in ("on", "serial") and comm_kind in ("loopback", "torch")
    if not split:
        overlap = "off"
    rw, cw, first = shard_windows(opts, p.A)
    plan = ShardPlan(p.A, G, row_window=rw, col_window=cw, first=first)
    if comm_kind in ("loopback", "loopback_fused"):
        comm = LoopbackComm(plan, fused=comm_kind == "loopback_fused")
        dev = torch.device("cuda", torch.cuda.current_device() if opts.device is None else opts.device)
        stream = torch.cuda.Stream(dev)
        shards = [DeviceLp(blk.A, blk.b, blk.c, opts, shard=blk, stream=stream)
                  for blk in (plan.block(g, p.A, p.b, p.c, local_first=split) for g in range(G))]
    elif comm_kind in ("torch", "torch_peer"):
        comm = TorchComm(plan, group, fused=comm_kind == "torch_peer")
        blk = plan.block(comm.rank, p.A, p.b, p.c, local_first=split)
        alloc = comm.symmetric_workspace if comm.fused else None
        shards = [DeviceLp(blk.A, blk.b, blk.c, opts, shard=blk, ws_alloc=alloc)]
    else:
        raise ValueError(comm_kind)
    if comm.fused:
        comm.connect_peers(shards)
    if hasattr(comm, "connect_fail"):
        comm.connect_fail(shards)   # loopback: same device; torch_peer: NVLink atomics
    return ShardedDevice(plan, shards, comm, overlap=overlap)


def run_pdhg_sharded(p, params=None, seed: int = 0, *, G: int, comm_kind: str = "loopback",
                     gpu=None, group=None, overlap: str = "auto"):
    """run_pdhg (pdhg.py:162-258) over G shards; same results contract."""
    import threading
    import time

    from . import engine
    from .lp_types import resolve

    T = resolve()
    opts = gpu or engine.GpuOptions()
    if params is None:
        params = T.PdhgParams()
    m, n = p.A.shape
    if m == 0 or n == 0:
        raise T.InvalidModelError("pdhg requires a nonempty model")
    t0 = time.monotonic()
    if p.A.nnz == 0:
        raise T.InvalidModelError("cannot estimate the norm of an empty matrix")
    dev = build_sharded(p, G, comm_kind, opts, group, overlap=overlap)
    dev.lock = threading.Lock()
    return engine._run(T, dev, p, params, seed, opts, t0)


# ------------------------------------------------- per-rank blocks (no full model)


def plan_state(plan: ShardPlan) -> dict:
    """What a rank needs of the plan without the matrix (cuts, slots, sizes)."""
    return {k: getattr(plan, k) for k in ("G", "m", "n", "nnz", "rcut", "ccut", "maxR", "maxC",
                                          "m_full", "n_full", "yslot", "xslot")}


def plan_from_state(state: dict) -> ShardPlan:
    plan = ShardPlan.__new__(ShardPlan)
    for k, v in state.items():
        setattr(plan, k, v)
    return plan


def save_block(path, plan: ShardPlan, blk: ShardBlock, b_full, c_full) -> None:
    """One rank's block + the plan's state, as an uncompressed .npz (e.g. under
    /dev/shm): ranks then load only their own rows instead of every rank
    generating and slicing the whole model."""
    arrays = {f"plan_{k}": np.asarray(v) for k, v in plan_state(plan).items()}
    for key, M in (("A", blk.A), ("At", blk.At)):
        arrays[f"{key}_data"], arrays[f"{key}_indices"] = M.data, M.indices
        arrays[f"{key}_indptr"], arrays[f"{key}_shape"] = M.indptr, np.asarray(M.shape)
    for k in ("b", "c"):
        arrays[k] = getattr(blk, k)
    for k in ("a_nloc", "at_nloc"):
        if getattr(blk, k) is not None:
            arrays[k] = getattr(blk, k)
    arrays["meta"] = np.asarray([blk.g, blk.m_full, blk.n_full, blk.y_off, blk.x_off])
    arrays["b_full"], arrays["c_full"] = np.asarray(b_full, float), np.asarray(c_full, float)
    np.savez(path, **arrays)


def load_block(path):
    """(plan, block, b_full, c_full) from save_block's file."""
    z = np.load(path)
    state = {k[len("plan_"):]: (z[k].item() if z[k].ndim == 0 else z[k]) for k in z.files
             if k.startswith("plan_")}
    plan = plan_from_state(state)
    mats = {key: sp.csr_matrix((z[f"{key}_data"], z[f"{key}_indices"], z[f"{key}_indptr"]),
                               shape=tuple(z[f"{key}_shape"])) for key in ("A", "At")}
    for M in mats.values():
        M.has_sorted_indices = False     # local-first blocks are not column-sorted
    g, m_full, n_full, y_off, x_off = (int(v) for v in z["meta"])
    blk = ShardBlock(g, mats["A"], mats["At"], z["b"], z["c"], m_full, n_full, y_off, x_off,
                     z["a_nloc"] if "a_nloc" in z.files else None,
                     z["at_nloc"] if "at_nloc" in z.files else None)
    return plan, blk, z["b_full"], z["c_full"]


def build_sharded_from_block(plan: ShardPlan, blk: ShardBlock, comm_kind: str = "torch", opts=None,
                             group=None, overlap: str = "auto", shard_factory=None):
    """This rank's ShardedDevice from its own block (torch.distributed job).
    ``shard_factory(blk)``: a stand-in shard backend (CPU tests' numpy double)."""
    from .engine import DeviceLp, GpuOptions

    opts = opts or GpuOptions()
    if comm_kind not in ("torch", "torch_peer"):
        raise ValueError("build_sharded_from_block is for one shard per process")
    comm = TorchComm(plan, group, fused=comm_kind == "torch_peer")
    if comm.rank != blk.g:
        raise ValueError(f"block {blk.g} loaded on rank {comm.rank}")
    if overlap == "auto":
        overlap = "on" if comm_kind == "torch" and blk.a_nloc is not None else "off"
    if overlap != "off" and blk.a_nloc is None:
        raise ValueError("the overlapped schedule needs a local_first block")
    alloc = comm.symmetric_workspace if comm.fused else None
    shards = [shard_factory(blk) if shard_factory is not None
              else DeviceLp(blk.A, blk.b, blk.c, opts, shard=blk, ws_alloc=alloc)]
    if comm.fused:
        comm.connect_peers(shards)
    return ShardedDevice(plan, shards, comm, overlap=overlap)


def run_pdhg_sharded_block(plan: ShardPlan, blk: ShardBlock, b_full, c_full, params=None, seed: int = 0, *,
                           comm_kind: str = "torch", gpu=None, group=None, overlap: str = "auto",
                           shard_factory=None):
    """run_pdhg (pdhg.py:162-258) from this rank's block; same results contract.
    The host loop reads only b and c of the whole model (its norms)."""
    import threading
    import time

    from . import engine
    from .lp_types import resolve

    T = resolve()
    opts = gpu or engine.GpuOptions()
    if params is None:
        params = T.PdhgParams()
    if plan.m == 0 or plan.n == 0:
        raise T.InvalidModelError("pdhg requires a nonempty model")
    t0 = time.monotonic()

    class _Model:   # what engine._run reads of the StandardLp
        pass

    p = _Model()
    p.b, p.c = np.asarray(b_full, float), np.asarray(c_full, float)
    dev = build_sharded_from_block(plan, blk, comm_kind, opts, group, overlap, shard_factory)
    dev.lock = threading.Lock()
    return engine._run(T, dev, p, params, seed, opts, t0)
