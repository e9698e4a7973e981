"""Multi-GPU host logic on CPU: shard plan, rank-order combine, and a
world_size-2 gloo run of the sharded engine (numpy shard doubles) against
the oracle.  The CUDA shards are exercised on the GPU in test_gpu_sharded.py."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch.multiprocessing as mp

import oracle
from conftest import load_golden
from oracle.pdhg_port import Model
from paper_2603_03150_b200 import _native as N
from paper_2603_03150_b200.sharded import ShardPlan, ShardedDevice, LoopbackComm, _combine


@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_shard_plan_reassembles_the_matrix(G):
    gm = load_golden("config0_s0")
    plan = ShardPlan(gm.A, G)
    assert plan.rcut[0] == 0 and plan.rcut[-1] == gm.m
    assert plan.ccut[0] == 0 and plan.ccut[-1] == gm.n
    assert np.all(np.diff(plan.rcut) >= 0) and np.all(np.diff(plan.ccut) >= 0)
    # slots are injective and monotone
    assert np.all(np.diff(plan.yslot) > 0) and np.all(np.diff(plan.xslot) > 0)
    assert plan.yslot.max() < plan.m_full and plan.xslot.max() < plan.n_full
    # the blocks, mapped back to original coordinates, are A and A'
    inv_x = np.full(plan.n_full, -1)
    inv_x[plan.xslot] = np.arange(gm.n)
    inv_y = np.full(plan.m_full, -1)
    inv_y[plan.yslot] = np.arange(gm.m)
    rows, cols = [], []
    trows, tcols = [], []
    nnz_per = []
    for g in range(G):
        blk = plan.block(g, gm.A, gm.b, gm.c)
        Ab = blk.A.tocoo()
        rows.append(Ab.row + plan.rcut[g])
        cols.append(inv_x[Ab.col])
        At = blk.At.tocoo()
        trows.append(At.row + plan.ccut[g])
        tcols.append(inv_y[At.col])
        nnz_per.append(blk.A.nnz)
        np.testing.assert_array_equal(blk.b, gm.b[plan.rcut[g]:plan.rcut[g + 1]])
        np.testing.assert_array_equal(blk.c, gm.c[plan.ccut[g]:plan.ccut[g + 1]])
    R = sp.coo_matrix((np.ones(sum(map(len, rows))), (np.concatenate(rows), np.concatenate(cols))),
                      shape=gm.A.shape).tocsr()
    assert (R != (gm.A != 0)).nnz == 0
    T = sp.coo_matrix((np.ones(sum(map(len, trows))), (np.concatenate(trows), np.concatenate(tcols))),
                      shape=(gm.n, gm.m)).tocsr()
    assert (T != (gm.A.T != 0)).nnz == 0
    # balanced: no shard holds much more than its share of entries
    assert max(nnz_per) <= gm.A.nnz / G + gm.A.getnnz(axis=1).max() + 1


def test_combine_is_rank_ordered_and_nan_propagating():
    rows = np.zeros((3, N.NQ))
    rows[:, N.Q_RP2] = [1e16, 1.0, -1e16]
    rows[:, N.Q_RPMAX] = [1.0, np.nan, 2.0]
    rows[:, N.Q_RDMAX] = [1.0, 3.0, 2.0]
    (q,) = _combine(rows, 1)
    assert q[N.Q_RP2] == ((1e16 + 1.0) + -1e16)
    assert np.isnan(q[N.Q_RPMAX])
    assert q[N.Q_RDMAX] == 3.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, eps, limit, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    from conftest import load_golden
    from paper_2603_03150_b200 import engine
    from paper_2603_03150_b200.lp_types import resolve
    from paper_2603_03150_b200.sharded import ShardPlan, ShardedDevice, TorchComm
    from shard_double import NumpyShard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gm = load_golden(name)
        plan = ShardPlan(gm.A, world)
        comm = TorchComm(plan)
        dev = ShardedDevice(plan, [NumpyShard(plan.block(rank, gm.A, gm.b, gm.c))], comm)
        T = resolve()
        pt, st = engine.run_on_device(dev, gm, T.PdhgParams(eps_rel=eps, max_kkt_passes=limit))
        q.put((rank, st.status.value, st.iterations, st.restarts, pt.x, pt.y, pt.z,
               st.termination.primal_lhs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,eps,limit", [("config0_s0", 1e-4, 200_000),
                                            ("eq_20x35_s17_ruiz", 1e-6, 200_000),
                                            ("eq_10x18_s7_ruiz", 1e-12, 200)])
def test_gloo_two_ranks_match_oracle(name, eps, limit):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, eps, limit, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gm = load_golden(name)
    opt, ost = oracle.run_pdhg(Model(gm.A, gm.b, gm.c),
                               oracle.PdhgParams(eps_rel=eps, max_kkt_passes=limit))
    (_, s0, it0, rs0, x0, y0, z0, pl0), (_, s1, it1, rs1, x1, y1, z1, pl1) = res
    # every rank took the same decisions and returns the same point
    assert (s0, it0, rs0) == (s1, it1, rs1)
    np.testing.assert_array_equal(x0, x1)
    np.testing.assert_array_equal(y0, y1)
    assert pl0 == pl1
    # and it is the reference's run (sums combined per shard: rounding only)
    assert s0 == ost.status.value
    assert it0 == ost.iterations and rs0 == ost.restarts
    np.testing.assert_allclose(x0, opt.x, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(y0, opt.y, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(z0, opt.z, rtol=1e-9, atol=1e-12)


def test_loopback_numpy_three_shards_match_oracle():
    """Loopback communicator over three numpy shards in one process."""
    from shard_double import NumpyShard

    from paper_2603_03150_b200 import engine
    from paper_2603_03150_b200.lp_types import resolve

    gm = load_golden("config0_s0")
    plan = ShardPlan(gm.A, 3)
    shards = [NumpyShard(plan.block(g, gm.A, gm.b, gm.c)) for g in range(3)]
    dev = ShardedDevice(plan, shards, LoopbackComm(plan))
    T = resolve()
    pt, st = engine.run_on_device(dev, gm, T.PdhgParams(eps_rel=1e-4))
    opt, ost = oracle.run_pdhg(Model(gm.A, gm.b, gm.c), oracle.PdhgParams(eps_rel=1e-4))
    assert st.iterations == ost.iterations and st.restarts == ost.restarts
    np.testing.assert_allclose(pt.x, opt.x, rtol=1e-9, atol=1e-12)


def failing_block_model():
    """config0_s0 beside an unbounded 2-column block (x1 = x2, c = -1e306):
    the last shard's x grows until it overflows at iteration 335 -- inside a
    64-iteration period -- while the other shards' iterates stay finite."""
    import scipy.sparse as sp

    gm = load_golden("config0_s0")
    A = sp.block_diag([gm.A, sp.csr_matrix(np.array([[1.0, -1.0]]))], format="csr")
    b = np.concatenate([gm.b, [0.0]])
    c = np.concatenate([gm.c, [-1e306, -1e306]])
    return Model(A, b, c)


@pytest.mark.parametrize("G", [2, 3])
def test_loopback_failure_stops_every_shard(G):
    """A non-finite iterate on one shard stops all shards at that iteration
    (connect_fail), so the sharded run returns the single-process failure point."""
    from shard_double import NumpyShard

    from paper_2603_03150_b200 import engine
    from paper_2603_03150_b200.lp_types import resolve

    p = failing_block_model()
    plan = ShardPlan(p.A, G)
    shards = [NumpyShard(plan.block(g, p.A, p.b, p.c)) for g in range(G)]
    comm = LoopbackComm(plan)
    comm.connect_fail(shards)
    dev = ShardedDevice(plan, shards, comm)
    T = resolve()
    pt, st = engine.run_on_device(dev, p, T.PdhgParams(eps_rel=1e-6, max_kkt_passes=500))
    opt, ost = oracle.run_pdhg(p, oracle.PdhgParams(eps_rel=1e-6, max_kkt_passes=500))
    assert ost.status.value == "NumericalFailure" and ost.iterations == 335
    assert st.status.value == ost.status.value and st.iterations == ost.iterations
    np.testing.assert_allclose(pt.x, opt.x, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(pt.y, opt.y, rtol=1e-9, atol=1e-12)
    assert [sh.fail for sh in shards] == [335] * G   # every shard stopped there


def _worker_time_limit(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    import time
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    from conftest import load_golden
    from paper_2603_03150_b200 import engine
    from paper_2603_03150_b200.lp_types import resolve
    from paper_2603_03150_b200.sharded import ShardPlan, ShardedDevice, TorchComm
    from shard_double import NumpyShard

    if rank == 1:   # this rank's clock jumps 1,000 s after the run starts
        real, calls = time.monotonic, [0]

        def late():
            calls[0] += 1
            return real() + (1000.0 if calls[0] > 1 else 0.0)

        engine.time.monotonic = late
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gm = load_golden("config0_s0")
        plan = ShardPlan(gm.A, world)
        dev = ShardedDevice(plan, [NumpyShard(plan.block(rank, gm.A, gm.b, gm.c))], TorchComm(plan))
        T = resolve()
        pt, st = engine.run_on_device(dev, gm, T.PdhgParams(eps_rel=1e-12, time_limit_s=500.0))
        q.put((rank, st.status.value, st.iterations))
    finally:
        dist.destroy_process_group()


def test_gloo_time_limit_is_collective():
    """One rank past the time limit stops every rank at the same iteration
    (ShardedDevice.agree) instead of leaving the others in a collective."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_time_limit, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == [(0, "TimeLimit", 0), (1, "TimeLimit", 0)]


def dense_row_model():
    """config0_s0 plus one dense linking row over every column (a budget row
    holding more than nnz/G entries): equal-nnz cuts would collide on it."""
    gm = load_golden("config0_s0")
    rng = np.random.default_rng(3)
    dense = sp.csr_matrix(rng.uniform(0.5, 1.5, (1, gm.n)))
    A = sp.vstack([dense, gm.A], format="csr")
    x0 = np.abs(rng.standard_normal(gm.n)) * (rng.random(gm.n) < 0.5)
    b = np.concatenate([dense @ x0, gm.b])
    return Model(A, b, gm.c.copy())


@pytest.mark.parametrize("G", [16, 24])
def test_shard_plan_dense_row_gives_no_empty_shard(G):
    p = dense_row_model()
    assert p.A.getnnz(axis=1)[0] >= 2 * p.A.nnz / G      # the dense row spans two cut targets
    plan = ShardPlan(p.A, G)
    assert np.all(np.diff(plan.rcut) >= 1) and np.all(np.diff(plan.ccut) >= 1)
    for g in range(G):
        blk = plan.block(g, p.A, p.b, p.c)
        assert blk.A.shape[0] >= 1 and blk.At.shape[0] >= 1


def test_shard_plan_rejects_more_shards_than_rows():
    A = sp.csr_matrix(np.ones((2, 5)))
    with pytest.raises(ValueError, match="cannot shard 2 rows over 3 shards"):
        ShardPlan(A, 3)


def test_loopback_dense_row_matches_oracle():
    """The sharded engine (16 numpy shards, loopback) on the dense-row model."""
    from shard_double import NumpyShard

    from paper_2603_03150_b200 import engine
    from paper_2603_03150_b200.lp_types import resolve

    p = dense_row_model()
    plan = ShardPlan(p.A, 16)
    shards = [NumpyShard(plan.block(g, p.A, p.b, p.c)) for g in range(16)]
    dev = ShardedDevice(plan, shards, LoopbackComm(plan))
    T = resolve()
    pt, st = engine.run_on_device(dev, p, T.PdhgParams(eps_rel=1e-4, max_kkt_passes=640))
    opt, ost = oracle.run_pdhg(p, oracle.PdhgParams(eps_rel=1e-4, max_kkt_passes=640))
    assert st.status.value == ost.status.value
    assert st.iterations == ost.iterations and st.restarts == ost.restarts
    np.testing.assert_allclose(pt.x, opt.x, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("G", [2, 3, 5])
def test_local_first_blocks(G):
    """local_first blocks: the same entries per row, the shard's own slot range
    first (a_nloc / at_nloc of them), each part in column order."""
    gm = load_golden("config0_s0")
    plan = ShardPlan(gm.A, G)
    for g in range(G):
        ref = plan.block(g, gm.A, gm.b, gm.c)
        blk = plan.block(g, gm.A, gm.b, gm.c, local_first=True)
        for M, R, nloc, lo, hi in ((blk.A, ref.A, blk.a_nloc, g * plan.maxC, (g + 1) * plan.maxC),
                                   (blk.At, ref.At, blk.at_nloc, g * plan.maxR, (g + 1) * plan.maxR)):
            np.testing.assert_array_equal(M.indptr, R.indptr)
            assert nloc.shape == (M.shape[0],)
            for r in range(M.shape[0]):
                s, e = M.indptr[r], M.indptr[r + 1]
                cols, vals = M.indices[s:e], M.data[s:e]
                k = int(nloc[r])
                assert np.all((cols[:k] >= lo) & (cols[:k] < hi))
                assert not np.any((cols[k:] >= lo) & (cols[k:] < hi))
                assert np.all(np.diff(cols[:k]) > 0) and np.all(np.diff(cols[k:]) > 0)
                order = np.argsort(cols, kind="stable")
                np.testing.assert_array_equal(cols[order], R.indices[s:e])
                np.testing.assert_array_equal(vals[order], R.data[s:e])


def _block_worker(rank, world, port, name, eps, limit, tmpdir, q):
    """One rank: loads ONLY its own block (written by rank 0 with save_block),
    runs the split-step schedule ("serial" on CPU) over gloo."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    from conftest import load_golden
    from paper_2603_03150_b200 import engine
    from paper_2603_03150_b200.lp_types import resolve
    from paper_2603_03150_b200.sharded import (ShardPlan, ShardedDevice, TorchComm, load_block,
                                               save_block)
    from shard_double import NumpyShard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        path = Path(tmpdir) / f"block_{rank}.npz"
        if rank == 0:
            gm = load_golden(name)
            plan = ShardPlan(gm.A, world)
            for g in range(world):
                save_block(Path(tmpdir) / f"block_{g}.npz", plan,
                           plan.block(g, gm.A, gm.b, gm.c, local_first=True), gm.b, gm.c)
            del gm, plan
        dist.barrier()
        plan, blk, b_full, c_full = load_block(path)
        assert blk.g == rank and blk.a_nloc is not None

        class P:
            pass

        p = P()
        p.b, p.c = b_full, c_full
        dev = ShardedDevice(plan, [NumpyShard(blk)], TorchComm(plan), overlap="on")
        assert dev.overlap == "serial"      # CPU doubles: no side stream
        T = resolve()
        pt, st = engine.run_on_device(dev, p, T.PdhgParams(eps_rel=eps, max_kkt_passes=limit))
        q.put((rank, st.status.value, st.iterations, st.restarts, pt.x, pt.y, pt.z))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,eps,limit", [("config0_s0", 1e-4, 200_000),
                                            ("eq_10x18_s7_ruiz", 1e-12, 200)])
def test_gloo_two_ranks_from_saved_blocks_split_schedule(name, eps, limit, tmp_path):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_block_worker, args=(r, 2, port, name, eps, limit, str(tmp_path), q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gm = load_golden(name)
    opt, ost = oracle.run_pdhg(Model(gm.A, gm.b, gm.c),
                               oracle.PdhgParams(eps_rel=eps, max_kkt_passes=limit))
    (_, s0, it0, rs0, x0, y0, z0), (_, s1, it1, rs1, x1, y1, z1) = res
    assert (s0, it0, rs0) == (s1, it1, rs1)
    np.testing.assert_array_equal(x0, x1)
    assert s0 == ost.status.value and it0 == ost.iterations and rs0 == ost.restarts
    np.testing.assert_allclose(x0, opt.x, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(y0, opt.y, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(z0, opt.z, rtol=1e-9, atol=1e-12)


def _bench_blocks_worker(rank, world, port, q):
    """bench.py's N>1 plumbing on CPU: rank 0 writes the per-rank blocks of a
    scaled config 4, every rank loads only its own and runs
    run_pdhg_sharded_block (numpy shard double, split schedule) over gloo."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    import types
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    import bench
    import paper_2603_03150_b200 as eng
    from paper_2603_03150_b200.sharded import run_pdhg_sharded_block
    from shard_double import NumpyShard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        args = types.SimpleNamespace(scale=0.0005, seed=4, ttk=False)
        blocks = bench._shard_blocks(args, world, rank, 0, eng, None)
        plan, blk, b, c = blocks["unscaled"]
        T = eng.types()
        pt, st = run_pdhg_sharded_block(plan, blk, b, c, T.PdhgParams(eps_rel=1e-12, max_kkt_passes=128),
                                        comm_kind="torch", overlap="on", shard_factory=NumpyShard)
        q.put((rank, blk.g, blk.A.shape[0], st.iterations, pt.x, pt.y, bench._host_rss_gb()))
    finally:
        dist.destroy_process_group()


def test_bench_block_files_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_blocks_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, g0, rows0, it0, x0, y0, rss0), (r1, g1, rows1, it1, x1, y1, rss1) = res
    assert (g0, g1) == (0, 1) and rows0 > 0 and rows1 > 0
    assert it0 == it1 == 128
    np.testing.assert_array_equal(x0, x1)
    from paper_2603_03150_b200.instances import config4

    inst = config4(scale=0.0005, seed=4)
    assert rows0 + rows1 == inst.m
    opt, ost = oracle.run_pdhg(Model(inst.A, inst.b, inst.c),
                               oracle.PdhgParams(eps_rel=1e-12, max_kkt_passes=128))
    np.testing.assert_allclose(x0, opt.x, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(y0, opt.y, rtol=1e-9, atol=1e-12)
    assert rss0 > 0 and rss1 > 0


def _fail_worker(rank, world, port, overlap, q):
    """gloo world: the NCCL-style all-gather mode, whose ranks do not share fail
    words -- a non-finite iterate on one rank must still stop every rank at
    the reference's iteration with the reference's failure-exit point."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    from paper_2603_03150_b200 import engine
    from paper_2603_03150_b200.lp_types import resolve
    from paper_2603_03150_b200.sharded import ShardPlan, ShardedDevice, TorchComm
    from shard_double import NumpyShard
    from test_sharded_cpu import failing_block_model

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = failing_block_model()
        plan = ShardPlan(p.A, world)
        sh = NumpyShard(plan.block(rank, p.A, p.b, p.c, local_first=overlap != "off"))
        dev = ShardedDevice(plan, [sh], TorchComm(plan), overlap=overlap)
        T = resolve()
        pt, st = engine.run_on_device(dev, p, T.PdhgParams(eps_rel=1e-6, max_kkt_passes=500))
        q.put((rank, st.status.value, st.iterations, pt.x, pt.y, pt.z, sh.fail,
               float(sh.v["xbar"].sum()), float(sh.v["ybar"].sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overlap", ["off", "on"])
def test_gloo_failure_stops_every_rank(overlap):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fail_worker, args=(r, 2, port, overlap, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    p = failing_block_model()
    opt, ost = oracle.run_pdhg(p, oracle.PdhgParams(eps_rel=1e-6, max_kkt_passes=500))
    assert ost.status.value == "NumericalFailure" and ost.iterations == 335
    for rank, status, its, x, y, z, fail, xbs, ybs in res:
        assert status == ost.status.value and its == ost.iterations
        np.testing.assert_allclose(x, opt.x, rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(y, opt.y, rtol=1e-9, atol=1e-12)
    # the rank that did not fail stopped at the failing iteration too: its running
    # averages are the single-process ones (checked against a loopback run with
    # shared fail words)
    from shard_double import NumpyShard

    from paper_2603_03150_b200 import engine
    from paper_2603_03150_b200.lp_types import resolve

    plan = ShardPlan(p.A, 2)
    shards = [NumpyShard(plan.block(g, p.A, p.b, p.c)) for g in range(2)]
    comm = LoopbackComm(plan)
    comm.connect_fail(shards)
    engine.run_on_device(ShardedDevice(plan, shards, comm), p,
                         resolve().PdhgParams(eps_rel=1e-6, max_kkt_passes=500))
    for (rank, *_, xbs, ybs), sh in zip(res, shards):
        assert xbs == pytest.approx(float(sh.v["xbar"].sum()), rel=1e-12, abs=1e-300, nan_ok=True)
        assert ybs == pytest.approx(float(sh.v["ybar"].sum()), rel=1e-12, abs=1e-300, nan_ok=True)


@pytest.mark.parametrize("first", [0, 32])
@pytest.mark.parametrize("G", [1, 2, 3])
def test_plan_row_window_renumbers_inside_blocks(G, first):
    """ShardPlan(row_window=..., col_window=...): every block keeps its rows
    and columns, each ordered by decreasing length inside each window; yslot /
    xslot map the originals to their slots, so the blocks reassemble A and A'
    exactly."""
    from paper_2603_03150_b200.instances import config4

    A = config4(0.001, seed=4).A
    w = 64
    plan = ShardPlan(A, G, row_window=w, col_window=w, first=first)
    base = ShardPlan(A, G)
    assert np.array_equal(plan.rcut, base.rcut) and plan.m_full == base.m_full
    lens = np.diff(A.indptr)
    inv_y = np.full(plan.m_full, -1)
    inv_y[plan.yslot] = np.arange(A.shape[0])
    inv_x = np.full(plan.n_full, -1)
    inv_x[plan.xslot] = np.arange(A.shape[1])
    rows, cols, vals, trows, tcols, tvals = [], [], [], [], [], []
    for g in range(G):
        blk = plan.block(g, A, np.arange(A.shape[0], dtype=float), np.arange(A.shape[1], dtype=float))
        r0, r1 = plan.rcut[g], plan.rcut[g + 1]
        orig = inv_y[g * plan.maxR + np.arange(r1 - r0)]
        assert sorted(orig) == list(range(r0, r1))                 # the block keeps its rows
        np.testing.assert_array_equal(blk.b, orig.astype(float))    # b follows the rows
        bl = lens[orig]
        _check_length_order(bl, lens[r0:r1], w, first)
        Ab = blk.A.tocoo()
        rows.append(orig[Ab.row]); cols.append(inv_x[Ab.col]); vals.append(Ab.data)
        c0, c1 = plan.ccut[g], plan.ccut[g + 1]
        ocol = inv_x[g * plan.maxC + np.arange(c1 - c0)]
        assert sorted(ocol) == list(range(c0, c1))                  # the block keeps its columns
        np.testing.assert_array_equal(blk.c, ocol.astype(float))    # c follows them
        cl = np.diff(blk.At.indptr)
        counts = np.bincount(A.indices, minlength=A.shape[1])
        np.testing.assert_array_equal(cl, counts[ocol])
        _check_length_order(cl, counts[c0:c1], w, first)
        At = blk.At.tocoo()                                          # rows: the block's columns
        trows.append(ocol[At.row])
        tcols.append(inv_y[At.col])
        tvals.append(At.data)
    R = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=A.shape)
    assert (R != A).nnz == 0
    T = sp.csr_matrix((np.concatenate(tvals), (np.concatenate(tcols), np.concatenate(trows))), shape=A.shape)
    assert (T != A).nnz == 0


def _check_length_order(new_lens, old_lens, w, first):
    """new_lens (block order after renumbering) against the block's natural
    lengths: with first = 0, decreasing inside every window of w; with
    first > 0, the long rows (> first) of every window first, each group
    keeping windows in order and decreasing length inside each window."""
    win = np.arange(old_lens.size) // w
    groups = [np.ones(old_lens.size, bool)] if first <= 0 else [old_lens > first, old_lens <= first]
    pos = 0
    for gmask in groups:
        for k in range(int(win[-1]) + 1 if old_lens.size else 0):
            sel = old_lens[gmask & (win == k)]
            got = new_lens[pos:pos + sel.size]
            np.testing.assert_array_equal(got, np.sort(sel)[::-1])
            pos += sel.size
    assert pos == old_lens.size
