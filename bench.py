"""Benchmark: PDHG iterations/s on BASELINE config 4 (5M x 10M, 200M nnz, fp64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scale S] [--ttk]

A *step* is one PDHG period: check_every=64 iterations (pdhg_step,
pdhg.py:140-151) followed by the KKT scoring of the current and averaged
iterates (pdhg.py:201-204) -- the unit in which run_pdhg talks to the device.
``value`` = iterations/s over K timed steps with the LP resident in HBM
(CUDA events on the engine's stream, max over ranks).  ``e2e`` = the same
metric through the public drop-in call ``run_pdhg(p, params)`` on host
arrays: layout upload + device transpose + power iteration + K*64
iterations + result download, all inside the timed region.

``--impl reference`` times the reference's own CPU implementation of the
path: the UNMODIFIED ``hybridlp`` package installed by ``oracle/make_ref.sh``
into oracle/_ref/site (its ``pdhg_step``, pdhg.py:140-151, and its two-point
``_score`` + ``check_relative_termination`` check, pdhg.py:201-204) on the
same instance, with OPENBLAS/OMP threads pinned to 1 (scipy's csr_matvec is
single-threaded).  A step is the same unit in both arms, one
period of 64 iterations plus the check; on the CPU it is extrapolated from a
bounded sample (K pdhg_step calls + one check), stated in
``cpu_baseline.sample``.  Without oracle/_ref (not built) it falls back to
the oracle port (oracle/pdhg_port.py, pinned bit-for-bit to the reference),
``kind: "port"``.

Inputs (4.8 GB of matrix) are far larger than the 126 MB L2, so no L2 flush
is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "PDHG iters/s and time-to-1e-4 rel KKT; achieved HBM GB/s vs B200 peak"
UNIT = "iter/s"
CHECK_EVERY = 64
NOMINAL_HBM_GBS = 8000.0   # north_star: "roughly 8 TB/s per B200"


def _config(m: int, n: int, nnz: int, scale: float, seed: int) -> dict:
    """The `config` object, identical in both arms (same instance, same step)."""
    return {"workload": f"config4 (m={m}, n={n}, nnz={nnz}) PDHG period = {CHECK_EVERY} iterations "
                        f"+ KKT check (pdhg.py:140-151, 198-204)",
            "scale": scale, "seed": seed,
            "l2": (f"no flush: {24 * nnz / 1e9:.1f} GB matrix (A and A') > 126 MB L2 (inputs larger than L2)"
                   if 24 * nnz > 4 * 126e6 else "no flush (small scaled instance; L2-resident)")}


def _cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _reference_ttk_iterations():
    """Iterations the REAL reference needed to reach 1e-4 on this instance
    (tests/golden/run_config4_s1[_nolimit].json, oracle/make_golden_runs.py;
    only a run that reached Optimal counts), or None."""
    for name in ("run_config4_s1_nolimit.json", "run_config4_s1.json"):
        try:
            r = json.loads((ROOT / "tests" / "golden" / name).read_text())
            if r.get("status") == "Optimal":
                return int(r["iterations"])
        except Exception:
            continue
    return None


def _env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return None


def _instance(scale: float, seed: int):
    from paper_2603_03150_b200.instances import config4

    return config4(scale=scale, seed=seed)


def live_kernel_ms(dev, it0: int, step: float, iters: int = 64) -> dict:
    """Average in-sequence duration (ms) of the primal and dual step kernels over
    one period launched kernel by kernel (pdhg_half_step) on the engine stream,
    an event pair around each launch."""
    import torch

    s = dev.stream
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(iters)] for _ in range(2)]
    dev.set_step(it0, step, step, float(it0))
    with torch.cuda.stream(s):
        for j in range(iters):
            for k, primal in ((0, True), (1, False)):
                a, b = ev[k][j]
                a.record(s)
                dev.half_step(primal, j)
                b.record(s)
    s.synchronize()
    return {name: sum(a.elapsed_time(b) for a, b in ev[k]) / iters
            for k, name in ((0, "primal"), (1, "dual"))}


def algorithmic_bytes(m: int, n: int, nnz: int) -> dict:
    """Bytes one PDHG iteration must move, fp64 values, int32 indices.

    primal step (rows of A'): 12 nnz + 4(n+1) offsets + 8m (y gather, compulsory)
                              + 24n (c, x, avg_x) + 24n (write x, xe, avg_x)
    dual step   (rows of A):  12 nnz + 4(m+1) offsets + 8n (xe gather, compulsory)
                              + 24m (b, y, avg_y) + 16m (write y, avg_y)
    total = 24 nnz + 60 n + 52 m (+8).
    check (every 64): A[x,avg_x] + A'[y,avg_y] = 24 nnz + 44 n + 44 m.
    """
    primal = 12 * nnz + 4 * (n + 1) + 8 * m + 48 * n
    dual = 12 * nnz + 4 * (m + 1) + 8 * n + 40 * m
    check = 24 * nnz + 44 * n + 44 * m
    return {"primal": primal, "dual": dual, "iter": primal + dual, "check": check}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/bench_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self) -> dict:
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = [r.split(",") for r in self.path.read_text().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) < 9:
                continue
            for k, nm in enumerate(names):
                if r[5 + k].strip().lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _pin_host_threads() -> None:
    """The reference path is single-threaded (scipy csr_matvec); pin BLAS and
    OpenMP to one thread for its norms/dots too.  Effective
    when called before numpy is first imported (the reference arm)."""
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"


def _reference_impl():
    """(module-like namespace, kind): the unmodified reference package from
    oracle/_ref/site when built (oracle/make_ref.sh), else the oracle port."""
    site = ROOT / "oracle" / "_ref" / "site"
    if (site / "hybridlp" / "pdhg.py").exists():
        if str(site) not in sys.path:
            sys.path.insert(0, str(site))
        import hybridlp
        from hybridlp import lp_core, pdhg

        if not str(Path(hybridlp.__file__).resolve()).startswith(str(site.resolve())):
            raise RuntimeError(f"hybridlp resolved outside oracle/_ref: {hybridlp.__file__}")

        class R:
            kind = "reference"
            where = "hybridlp (unmodified reference, oracle/_ref/site)"
            model = staticmethod(lambda A, b, c: lp_core.StandardLp(A, b, c))
            step = staticmethod(pdhg.pdhg_step)
            score = staticmethod(pdhg._score)
            term = staticmethod(lp_core.check_relative_termination)
            State = pdhg.PdhgState
        return R
    import oracle
    from oracle.pdhg_port import Model, PdhgState, _score, check_relative_termination

    class P:
        kind = "port"
        where = "oracle/pdhg_port.py (reference restated, pinned bit-for-bit)"
        model = staticmethod(Model)
        step = staticmethod(oracle.pdhg_step)
        score = staticmethod(_score)
        term = staticmethod(check_relative_termination)
        State = PdhgState
    return P


def cpu_sample(inst, steps: int = 3, warmup: int = 1) -> dict:
    """The reference's CPU path on `inst`: `steps` timed pdhg_step calls (after
    `warmup` untimed ones) and one two-point check (pdhg.py:201-204), i.e. one
    period = 64 steps + 1 check, extrapolated from the sample."""
    import numpy as np

    R = _reference_impl()
    p = R.model(inst.A, inst.b, inst.c)
    t = time.perf_counter()
    p.A_csc  # the reference builds its CSC copy lazily on first at_y (lp_core.py:133-138)
    t_csc = time.perf_counter() - t
    st = R.State(x=np.zeros(p.n), y=np.zeros(p.m), avg_x=np.zeros(p.n), avg_y=np.zeros(p.m),
                 avg_weight=0.0, tau=0.5 / 40.0, sigma=0.5 / 40.0, omega=1.0, iterations=0,
                 restarts=0, restart_x=None, restart_y=None, restart_score=1.0)
    for _ in range(max(1, warmup)):
        R.step(st, p)
    samples = []
    for _ in range(steps):
        t = time.perf_counter()
        R.step(st, p)
        samples.append(time.perf_counter() - t)
    t = time.perf_counter()
    cur_pt, _, _ = R.score(p, st.x, st.y)
    avg_pt, _, _ = R.score(p, st.avg_x, st.avg_y)
    R.term(p, cur_pt, 1e-4)
    R.term(p, avg_pt, 1e-4)
    t_check = time.perf_counter() - t
    t_step = sum(samples) / len(samples)
    per_iter = t_step + t_check / CHECK_EVERY
    return {"per_iter_s": per_iter, "step_s": t_step, "check_s": t_check, "tocsc_s": t_csc,
            "steps": steps, "step_s_samples": samples, "kind": R.kind, "impl": R.where}


def _cpu_baseline(cs: dict, m: int, n: int, nnz: int) -> dict:
    value = 1.0 / cs["per_iter_s"]
    ref_its = _reference_ttk_iterations()
    out = {"value": value, "unit": UNIT, "cores": 1, "kind": cs["kind"],
           "sample": (f"{cs['impl']} on the same config4 instance (m={m}, n={n}, nnz={nnz}): "
                      f"{cs['steps']} timed pdhg_step calls ({cs['step_s']:.3f} s each) + one two-point "
                      f"check ({cs['check_s']:.2f} s) amortised over {CHECK_EVERY} iterations; "
                      f"OPENBLAS/OMP threads = 1 (scipy csr_matvec is single-threaded)"),
           "host": {"cpu_model": _cpu_model(), "nproc": os.cpu_count(), "active_cores": 1},
           "ms_per_period": (CHECK_EVERY * cs["step_s"] + cs["check_s"]) * 1e3}
    if ref_its:
        out["time_to_1e4_s"] = {"value": ref_its * cs["per_iter_s"], "iterations": ref_its,
                                "note": "extrapolated: iterations the real reference took to reach 1e-4 "
                                        "on this instance (tests/golden/run_config4_s1_nolimit.json) x the "
                                        "sampled seconds per iteration"}
    return out


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return 0
    _pin_host_threads()
    inst = _instance(args.scale, args.seed)
    cs = cpu_sample(inst, steps=args.steps, warmup=args.warmup)
    cpu = _cpu_baseline(cs, inst.m, inst.n, inst.nnz)
    value = cpu["value"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": cpu["ms_per_period"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": _config(inst.m, inst.n, inst.nnz, args.scale, args.seed),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_s_samples": cs["step_s_samples"], "check_s": cs["check_s"],
    }
    print(json.dumps(line))
    return 0


def _shard_blocks(args, world: int, rank: int, local: int, eng, opts) -> dict:
    """Rank 0: generate config 4, equilibrate it on its GPU (device Ruiz), cut
    both into local-first per-rank blocks (sharded.ShardPlan) and write them to
    /dev/shm; every rank: load only its own two blocks.  Returns the loaded
    (plan, block, b, c) pairs and rank 0's Ruiz time."""
    import shutil

    import torch
    import torch.distributed as dist

    from paper_2603_03150_b200.sharded import ShardPlan, load_block, save_block, shard_windows

    need = 2 * 30e9 * max(args.scale, 0.01)          # both models' blocks (~24 B/entry + vectors)
    root = Path("/dev/shm")
    if not root.is_dir() or shutil.disk_usage(root).free < need:
        root = Path(os.environ.get("TMPDIR", "/tmp"))
    shm = root / f"pdhg_bench_{os.environ.get('MASTER_PORT', '0')}"
    meta = [None]
    if rank == 0:
        shm.mkdir(parents=True, exist_ok=True)
        inst = _instance(args.scale, args.seed)
        for tag, model in (("unscaled", inst), ("scaled", None)):
            if model is None:
                if not args.ttk:
                    break
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                model, info = eng.ruiz_equilibrate(inst, gpu=opts, register_layout=False)
                torch.cuda.synchronize()
                meta[0] = {"ruiz_s": time.perf_counter() - t0, "ruiz_passes": info.applied_iterations,
                           "ruiz_phases": dict(eng.ruiz.last_timings)}
            rw, cw, first = shard_windows(opts, model.A)
            plan = ShardPlan(model.A, world, row_window=rw, col_window=cw, first=first)
            for g in range(world):
                save_block(shm / f"{tag}_{g}.npz", plan,
                           plan.block(g, model.A, model.b, model.c, local_first=True), model.b, model.c)
            del plan
        del inst
        if torch.cuda.is_available():
            torch.cuda.empty_cache()
    dist.broadcast_object_list(meta, src=0)
    out = {"unscaled": load_block(shm / f"unscaled_{rank}.npz")}
    if args.ttk:
        out["scaled"] = load_block(shm / f"scaled_{rank}.npz")
        out.update(meta[0])
    dist.barrier()
    if rank == 0:
        shutil.rmtree(shm, ignore_errors=True)
    return out


def _host_rss_gb() -> float:
    import resource

    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6   # KB -> GB (Linux)


def _allgather_ms(dev, reps: int = 32) -> dict:
    """Average time of the per-iteration all-gathers of xe and y alone (CUDA
    events on the shard stream), i.e. the exchange the overlap hides."""
    import torch

    s = dev.shards[0].stream
    out = {}
    for name in ("xe", "y"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            dev.comm.allgather(dev.shards, name)
            e0.record(s)
            for _ in range(reps):
                dev.comm.allgather(dev.shards, name)
            e1.record(s)
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / reps
    return out


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = _env_rank()
    # --sharded: the N > 1 path (rank-0 block files, sharded engine, NCCL
    # all-gathers, overlap schedule) also on a world of one -- a smoke test of
    # the multi-GPU bench on a one-GPU box, not a measurement
    sharded = world > 1 or args.sharded
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
    torch.cuda.set_device(local)
    if sharded:
        import datetime

        # rank 0 generates and cuts the 200M-entry model while the others wait
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(minutes=30))
    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200 import _native as N

    T = eng.types()
    opts = eng.GpuOptions(cache_layout=False, psr=args.psr)
    comm_kind = "torch_peer" if args.comm == "peer" else "torch"
    blocks = None
    if sharded:
        # rank 0 generates the LP (and its device-Ruiz-scaled twin for the run to
        # 1e-4), cuts it into per-rank blocks and writes them to /dev/shm; every
        # rank then holds only its own rows (no per-rank copy of the whole model)
        blocks = _shard_blocks(args, world, rank, local, eng, opts)
        plan, blk, b_full, c_full = blocks["unscaled"]
        m, n, nnz = plan.m, plan.n, plan.nnz
        inst = None
    else:
        inst = _instance(args.scale, args.seed)
        m, n, nnz = inst.m, inst.n, inst.nnz
    ab = algorithmic_bytes(m, n, nnz)

    # ---- device-resident timing: K periods of 64 iterations + check
    t_setup = time.perf_counter()
    if sharded:
        from paper_2603_03150_b200.sharded import build_sharded_from_block

        dev = build_sharded_from_block(plan, blk, comm_kind, opts, overlap=args.overlap)
        kdev = dev.shards[0]   # this rank's shard context (kernel timing)
    else:
        dev = kdev = eng.DeviceLp(inst.A, inst.b, inst.c, opts)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    rng = np.random.default_rng(0)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    lam = dev.opnorm(v)
    step = 1.0 / (1.05 * lam)
    dev.reset()
    it = 0
    # engine._run hands each two-point check's A'y of the current point to the
    # next period's first primal step when nothing restarts (check_dot)
    reuse = (lambda: dev.use_check_dot(0)) if getattr(dev, "check_dot", False) else (lambda: None)
    period = getattr(dev, "run_period_check", None)
    check_fused = bool(period is not None and getattr(dev, "check_fuse", False))
    for _ in range(args.warmup):   # the timed loop's own calls (graphs captured here)
        if period is not None:
            period(CHECK_EVERY, it, step, step, float(it), N.PT_CUR, N.PT_AVG)
        else:
            dev.run_period(CHECK_EVERY, it, step, step, float(it))
            dev.check(N.PT_CUR, N.PT_AVG)
        reuse()
        it += CHECK_EVERY
    s = kdev.stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if sharded:
        dist.barrier()
    torch.cuda.synchronize()
    # the product's period call (engine._run): the graph of 64 iterations and
    # the two-point check, one host synchronisation per period (with check_fuse
    # the check's A side runs inside the period's last dual step)
    with ClockSampler(local) as clk:
        ev0.record(s)
        for _ in range(args.steps):
            if period is not None:
                fail, _ = period(CHECK_EVERY, it, step, step, float(it), N.PT_CUR, N.PT_AVG)
            else:
                fail = dev.run_period(CHECK_EVERY, it, step, step, float(it))
                dev.check(N.PT_CUR, N.PT_AVG)
            reuse()
            it += CHECK_EVERY
        ev1.record(s)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    # where a period's time goes (after the timed region, same sustained state):
    # events around the graph of 64 iterations and around the check
    breakdown = None
    if not sharded:
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(3)]
        for e in evs:
            e[0].record(s)
            dev.run_period(CHECK_EVERY, it, step, step, float(it))
            e[1].record(s)
            dev.check(N.PT_CUR, N.PT_AVG)
            e[2].record(s)
            reuse()
            it += CHECK_EVERY
        pc = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(3)]
        if period is not None:
            for e in pc:
                e[0].record(s)
                period(CHECK_EVERY, it, step, step, float(it), N.PT_CUR, N.PT_AVG)
                e[1].record(s)
                reuse()
                it += CHECK_EVERY
        torch.cuda.synchronize()
        g_ms = [e[0].elapsed_time(e[1]) for e in evs]
        c_ms = [e[1].elapsed_time(e[2]) for e in evs]
        breakdown = {"graph_64_iterations_ms": statistics.median(g_ms),
                     "check_ms": statistics.median(c_ms),
                     "method": "3 periods after the timed region: CUDA events around the period graph "
                               "and around the two-point check (run_period + check, 2 host syncs)"}
        if period is not None:
            breakdown["period_check_ms"] = statistics.median(e[0].elapsed_time(e[1]) for e in pc)
            breakdown["check_fused"] = check_fused
            breakdown["method"] += ("; period_check_ms: 3 more periods through the product's "
                                    "run_period_check (check_fused: its A side inside the last dual step)")
    if sharded:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    iters = args.steps * CHECK_EVERY
    value = iters / (ms / 1e3)   # iterations of the one LP per second, all ranks together
    ms_per_step = ms / args.steps
    if sharded:   # kernel roofline below is for this rank's shard
        ab = algorithmic_bytes(kdev.m, kdev.n, kdev.nnz)
        ab["primal"] = 12 * kdev.at_nnz + 4 * (kdev.n + 1) + 8 * kdev.m_full + 48 * kdev.n
        ab["dual"] = 12 * kdev.nnz + 4 * (kdev.m + 1) + 8 * kdev.n_full + 40 * kdev.m

    # ---- per-kernel timing for the roofline (CUDA events on the engine stream)
    reps = 20
    if not sharded:
        # live: one more period right after the timed region, in the same
        # sustained (power-capped) state, launched kernel by kernel with an
        # event pair around every launch -- the in-sequence duration of each
        # step kernel as the graph runs it
        live_it = it
        tk = live_kernel_ms(kdev, live_it, step)
        tk_isolated = {"primal": kdev.time_kernel(0, reps, step, step),
                       "dual": kdev.time_kernel(1, reps, step, step)}
    else:
        tk = {"primal": kdev.time_kernel(0, reps, step, step), "dual": kdev.time_kernel(1, reps, step, step)}
        tk_isolated = dict(tk)
    comm_info = None
    if sharded:
        ag = _allgather_ms(dev)
        comm_info = {"overlap": dev.overlap, "comm": comm_kind,
                     "allgather_ms_per_iteration": {"xe": ag["xe"], "y": ag["y"], "sum": ag["xe"] + ag["y"]},
                     "allgather_bytes_received_per_rank": 8 * (plan.n_full + plan.m_full) * (world - 1) // world,
                     "pass0_entries_fraction": {
                         "A": float(blk.a_nloc.sum()) / max(1, blk.A.nnz) if blk.a_nloc is not None else None,
                         "At": float(blk.at_nloc.sum()) / max(1, blk.At.nnz) if blk.at_nloc is not None else None},
                     "method": "32 all-gathers of each vector alone, CUDA events on the shard stream (rank 0)"}
    top = max(tk, key=tk.get)
    peaks = _peaks()
    peak = peaks["hbm_gbs"] if peaks else 6650.0
    achieved = ab[top] / (tk[top] * 1e-3) / 1e9
    traffic = units = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        try:
            tj = json.loads(tf.read_text())
            traffic, units = tj.get(top), tj.get(f"{top}_units")
        except Exception:
            traffic = units = None
    iter_ms = ms_per_step / CHECK_EVERY
    roofline = {"bound": "hbm", "kernel": f"k_step<{'primal' if top == 'primal' else 'dual'}>",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "frac_nominal": achieved / NOMINAL_HBM_GBS,
                "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s",
                "kernels_ms": tk, "kernels_ms_method": (
                    "average of 64 in-sequence launches each, CUDA events on the engine stream, "
                    "one period launched kernel by kernel right after the timed region"
                    if not sharded else "pdhg_time_kernel: 20 repeated launches, CUDA events"),
                "kernels_ms_isolated": tk_isolated, "algorithmic_bytes": ab,
                # the units that bind (ncu capture, profiles/traffic.json): every gather of the
                # 40/80 MB vector is a 32 B L2 sector, so L1TEX / L2-slice throughput, not DRAM,
                # caps the step kernels
                "binding_units_pct_ncu": units,
                # the same kernel's frac at the clock ncu ran it (no power cap; informational --
                # `frac` above is the in-sequence, power-capped one this run measured)
                "frac_at_ncu_clock": (ab[top] / (units["time_us"] * 1e-6) / 1e9 / peak
                                      if units and units.get("time_us") else None),
                "iteration_gbs": (ab["iter"] + ab["check"] / CHECK_EVERY) / (iter_ms * 1e-3) / 1e9}
    # the timing leg's device memory goes back to torch's caching allocator
    # (not to the driver): the e2e call below reuses it, as repeated calls in
    # one serving process do (reported as e2e.allocator)
    def _op_layout(key, lanes):
        if getattr(kdev, "_psr", {}).get(key):
            return "psr"
        if getattr(kdev, "_sell_part", {}).get(key):
            return "sliced-ELL split (pass 0 local-slot entries, pass 1 the rest)"
        if getattr(kdev, "_sell", {}).get(key):
            return "sliced-ELL"
        split = getattr(kdev, "split_local", {}).get(key) is not None
        return f"csr-vector ({lanes} lanes/row)" + (" split" if split else "")

    layout_name = {"A (dual step)": _op_layout("A", kdev.a_lanes),
                   "A' (primal step)": _op_layout("At", kdev.at_lanes)}
    del dev, kdev, period    # (the bound method would keep the timing leg's layout alive)

    # ---- e2e through the public drop-in call, host arrays in, host arrays out
    K = args.steps
    params = T.PdhgParams(eps_rel=1e-12, max_kkt_passes=K * CHECK_EVERY)
    # each call is a whole solve from host arrays (fresh layout, cache_layout
    # off); --e2e-reps calls, the median is reported (the first pays whatever
    # device allocations the caching allocator cannot serve from its pool)
    e2e_runs = []
    for _ in range(max(1, args.e2e_reps)):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        if sharded:
            from paper_2603_03150_b200.sharded import run_pdhg_sharded_block

            # the public entry from this rank's host block (upload, layout, power
            # iteration, K*64 iterations, download), every rank at once
            pt, st = run_pdhg_sharded_block(plan, blk, b_full, c_full, params, gpu=opts,
                                            comm_kind=comm_kind, overlap=args.overlap)
        else:
            pt, st = eng.run_pdhg(inst, params, gpu=opts)
        e1.record()
        torch.cuda.synchronize()
        wall_e2e = time.perf_counter() - t0
        e2e_ms = e0.elapsed_time(e1)
        if sharded:
            t = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e_runs.append((st.iterations / (e2e_ms / 1e3), wall_e2e, st))
        del pt
    e2e_runs_sorted = sorted(e2e_runs, key=lambda r: r[0])
    e2e_value, wall_e2e, st = e2e_runs_sorted[len(e2e_runs_sorted) // 2]
    h2d = 12 * nnz + 4 * (m + 1) + 8 * (m + n) + 8 * n
    d2h = 8 * (2 * n + m)

    out = None
    if args.ttk:
        # the reference pipeline equilibrates before PDHG (prepare_model,
        # warmstart.py:178-197): device Ruiz, then run_pdhg on the scaled model
        # (its device layout is handed over, no second upload).  At N > 1 every
        # rank equilibrates the whole model (bit-identical), then the sharded
        # run; times are the max over ranks.
        ttk_params = T.PdhgParams(eps_rel=1e-4, time_limit_s=args.ttk_limit)
        if sharded:
            from paper_2603_03150_b200.sharded import run_pdhg_sharded_block

            splan, sblk, sb, sc = blocks["scaled"]
            t_ruiz, passes = blocks["ruiz_s"], blocks["ruiz_passes"]
            pt2, st2 = run_pdhg_sharded_block(splan, sblk, sb, sc, ttk_params, gpu=opts,
                                              comm_kind=comm_kind, overlap=args.overlap)
            tt = torch.tensor([st2.wall_seconds], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            wall2 = float(tt[0])

            class _I:
                applied_iterations = passes
            info = _I()
        else:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            scaled, info = eng.ruiz_equilibrate(inst, gpu=opts, register_layout=True)
            torch.cuda.synchronize()
            t_ruiz = time.perf_counter() - t0
            pt2, st2 = eng.run_pdhg(scaled, ttk_params, gpu=opts)
            wall2 = st2.wall_seconds
        out = {"status": st2.status.value, "iterations": st2.iterations, "restarts": st2.restarts,
               "pdhg_wall_s": wall2, "ruiz_s": t_ruiz, "ruiz_passes": info.applied_iterations,
               "total_s": t_ruiz + wall2,
               "ruiz_phases_s": dict(eng.ruiz.last_timings) if not sharded else blocks.get("ruiz_phases"),
               "reference_iterations": _reference_ttk_iterations(),
               "note": "device Ruiz (bit-identical to transform.py:35-77) + run_pdhg to eps_rel=1e-4"
                       + (f", sharded over {world} GPUs (Ruiz once on rank 0's GPU, blocks to "
                          f"/dev/shm)" if sharded else "")}
        if args.ttk_unscaled and not sharded:
            pt3, st3 = eng.run_pdhg(inst, T.PdhgParams(eps_rel=1e-4, time_limit_s=args.ttk_limit), gpu=opts)
            out["unscaled"] = {"status": st3.status.value, "iterations": st3.iterations,
                               "restarts": st3.restarts, "wall_s": st3.wall_seconds}

    cpu = None
    if rank == 0 and not sharded and not args.no_cpu:
        cs = cpu_sample(inst, steps=args.cpu_steps)
        cpu = _cpu_baseline(cs, m, n, nnz)
        if "time_to_1e4_s" not in cpu and out is not None and out.get("status") == "Optimal":
            its = int(out["iterations"])
            cpu["time_to_1e4_s"] = {"value": its * cs["per_iter_s"], "iterations": its,
                                    "note": "extrapolated: this run's GPU iteration count to 1e-4 x the "
                                            "reference's sampled seconds per iteration (the reference's "
                                            "own count, once tests/golden/run_config4_s1_nolimit.json exists)"}
    rss_max = _host_rss_gb()
    if sharded:
        t = torch.tensor([rss_max], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rss_max = float(t.item())
    if rank != 0:
        if sharded:
            dist.destroy_process_group()
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(m, n, nnz, args.scale, args.seed),
        "layout": {"parallelism": ((f"A rows / A' rows sharded x{world}, equal nnz; " +
                                    ("xe / y pushed to peers by the step epilogues (symmetric memory, "
                                     "NVLink stores) + stream barrier" if args.comm == "peer" else
                                     "NCCL all-gather of xe and y per iteration"))
                                   if sharded else "1 GPU"),
                   "kernel_layout": layout_name},
        "roofline": roofline,
        "period_breakdown": breakdown,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / K,
                "d2h_bytes_per_step": d2h / K, "iterations": st.iterations,
                "wall_s": wall_e2e, "timings": getattr(st, "timings", None),
                "runs_iter_s": [round(r[0], 2) for r in e2e_runs],
                "note": f"run_pdhg(StandardLp on host) incl. upload, transpose, opnorm; median of "
                        f"{len(e2e_runs)} calls",
                "allocator": "warm: torch caching allocator holds the timing leg's freed device blocks"},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        # per step: 2 step kernels per iteration (4 with the split steps of the
        # overlapped multi-GPU schedule) + the check's k_pair x2,
        # k_check_primal(_sell), k_check_dual(_sell), k_reduce; with the fused
        # check k_pair (y), k_check_primal_fold, k_check_dual_sell, k_reduce
        # (ncu launch list, profiles/r02_fa_launches.csv)
        "gpu_launches": args.steps * ((4 if comm_info and comm_info["overlap"] != "off" else 2)
                                      * CHECK_EVERY + (4 if check_fused else 5)),
        "setup_s": t_setup,
        "time_to_1e4": out,
        "multi_gpu": comm_info,
        "host_rss_gb_max_over_ranks": rss_max,
    }
    print(json.dumps(line))
    if sharded:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=4)
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--sharded", action="store_true",
                    help="run the multi-GPU (sharded, NCCL) path even on one GPU (smoke test)")
    ap.add_argument("--e2e-reps", type=int, default=3, help="public-API calls for e2e (median reported)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ttk", action=argparse.BooleanOptionalAction, default=True,
                    help="also run to eps_rel=1e-4 (time-to-1e-4, part of the metric; --no-ttk skips)")
    ap.add_argument("--ttk-limit", type=float, default=300.0)
    ap.add_argument("--ttk-unscaled", action="store_true", help="also run to 1e-4 without Ruiz")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "peer"],
                    help="N>1: all-gather xe/y with NCCL after each half step, or push them "
                         "from the step epilogues to the peers' symmetric memory")
    ap.add_argument("--overlap", default="auto", choices=["auto", "on", "serial", "off"],
                    help="N>1 NCCL mode: split half steps with the all-gather overlapping pass 0 "
                         "(on/auto), the same split kernels in line (serial), or unsplit (off)")
    ap.add_argument("--psr", default="off", choices=["off", "on", "auto"],
                    help="step-kernel layout (off = CSR-vector, the measured fastest)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
