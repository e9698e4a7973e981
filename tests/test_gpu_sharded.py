"""Sharded (multi-GPU) data path on one GPU: G CUDA shard contexts driven in
loopback (all-gather = device copies).  Exercises the padded-slot layouts,
slice-offset kernels, sharded power iteration and the rank-order combine of
per-shard check partials against the oracle."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import EXPERIMENTAL_BUILD, load_golden, skip_unless_experimental
from oracle.pdhg_port import KktPoint, Model

PSR_PARAMS = ["off", "on"] if EXPERIMENTAL_BUILD else ["off"]

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import paper_2603_03150_b200 as eng

    return eng


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("name,eps,limit", [("config0_s0", 1e-4, 200_000),
                                            ("eq_20x35_s17_ruiz", 1e-6, 200_000),
                                            ("ineq_12x20_s32_ruiz", 1e-4, 200_000),
                                            ("eq_10x18_s7_ruiz", 1e-12, 128)])
@pytest.mark.parametrize("psr", PSR_PARAMS)
def test_loopback_shards_match_reference(eng, G, name, eps, limit, psr):
    from paper_2603_03150_b200.sharded import run_pdhg_sharded

    if psr == "on":
        skip_unless_experimental("psr")
    gm = load_golden(name)
    T = eng.types()
    opts = eng.GpuOptions(psr=psr, psr_min_staged=1)
    pt, st = run_pdhg_sharded(gm, T.PdhgParams(eps_rel=eps, max_kkt_passes=limit), G=G, gpu=opts)
    r = gm.run({1e-4: "e4", 1e-6: "e6", 1e-12: "lim128"}[eps])
    assert st.status.value == str(r["status"])
    assert st.iterations == int(r["iterations"])
    assert st.restarts == int(r["restarts"])
    assert float(gm.c @ pt.x) == pytest.approx(float(r["obj"]), rel=1e-6, abs=1e-9)
    if st.status.value == "Optimal":
        t = oracle.check_relative_termination(Model(gm.A, gm.b, gm.c), KktPoint(pt.x, pt.y, pt.z), eps)
        assert t.ok
    else:
        np.testing.assert_allclose(pt.x, r["x"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(pt.y, r["y"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(pt.z, r["z"], rtol=1e-9, atol=1e-12)


def test_loopback_scaled_config4_matches_single_gpu(eng):
    from paper_2603_03150_b200.instances import config4
    from paper_2603_03150_b200.sharded import run_pdhg_sharded

    p = config4(scale=0.01, seed=21)  # 50k x 100k, ~2M nnz
    T = eng.types()
    pt1, st1 = eng.run_pdhg(p, T.PdhgParams(eps_rel=1e-4))
    pt4, st4 = run_pdhg_sharded(p, T.PdhgParams(eps_rel=1e-4), G=4)
    assert st1.status.value == st4.status.value == "Optimal"
    assert abs(st4.iterations - st1.iterations) <= 0.05 * st1.iterations
    assert float(p.c @ pt4.x) == pytest.approx(float(p.c @ pt1.x), rel=1e-6)
    t = oracle.check_relative_termination(Model(p.A, p.b, p.c), KktPoint(pt4.x, pt4.y, pt4.z), 1e-4)
    assert t.ok


def test_sharded_opnorm_matches(eng):
    from paper_2603_03150_b200.sharded import build_sharded

    gm = load_golden("config0_s0")
    dev = build_sharded(gm, 3)
    rng = np.random.default_rng(0)
    v = rng.standard_normal(gm.n)
    v /= np.linalg.norm(v)
    assert dev.opnorm(v) == pytest.approx(float(gm.g["opnorm_seed0"]), rel=1e-12)


def test_torch_comm_over_nccl_world1(eng):
    """The one-process-per-GPU path (TorchComm over NCCL) on a world of one:
    exercises the torch views of the library's vectors, the NCCL
    all_gather_into_tensor calls on the engine's stream and the rank-order
    combine, against the golden reference run."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2603_03150_b200.sharded import run_pdhg_sharded

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        gm = load_golden("config0_s0")
        T = eng.types()
        pt, st = run_pdhg_sharded(gm, T.PdhgParams(eps_rel=1e-4), G=1, comm_kind="torch")
        r = gm.run("e4")
        assert st.status.value == "Optimal"
        assert st.iterations == int(r["iterations"]) and st.restarts == int(r["restarts"])
        assert float(gm.c @ pt.x) == pytest.approx(float(r["obj"]), rel=1e-6)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("psr", PSR_PARAMS)
def test_fused_allgather_matches_copy_allgather(eng, G, psr):
    """Fused all-gather (epilogue peer stores, pdhg_set_peers) vs the all-gather
    after each half step: the same arithmetic, so bitwise-identical results."""
    from paper_2603_03150_b200.sharded import run_pdhg_sharded

    if psr == "on":
        skip_unless_experimental("psr")
    gm = load_golden("config0_s0")
    T = eng.types()
    opts = eng.GpuOptions(psr=psr, psr_min_staged=1)
    params = T.PdhgParams(eps_rel=1e-4)
    pa, sa = run_pdhg_sharded(gm, params, G=G, gpu=opts, comm_kind="loopback")
    pb, sb = run_pdhg_sharded(gm, params, G=G, gpu=opts, comm_kind="loopback_fused")
    assert (sa.status, sa.iterations, sa.restarts) == (sb.status, sb.iterations, sb.restarts)
    assert pa.x.tobytes() == pb.x.tobytes() and pa.y.tobytes() == pb.y.tobytes()
    assert pa.z.tobytes() == pb.z.tobytes()
    r = gm.run("e4")
    assert sb.iterations == int(r["iterations"]) and sb.restarts == int(r["restarts"])


def test_fused_allgather_scaled_config4(eng):
    """4 fused shards on a 2M-nnz config-4 instance reproduce the copy path bit for bit."""
    from paper_2603_03150_b200.instances import config4
    from paper_2603_03150_b200.sharded import run_pdhg_sharded

    p = config4(scale=0.01, seed=21)
    T = eng.types()
    params = T.PdhgParams(eps_rel=1e-12, max_kkt_passes=256)
    pa, sa = run_pdhg_sharded(p, params, G=4, comm_kind="loopback")
    pb, sb = run_pdhg_sharded(p, params, G=4, comm_kind="loopback_fused")
    assert sa.iterations == sb.iterations == 256
    assert pa.x.tobytes() == pb.x.tobytes() and pa.y.tobytes() == pb.y.tobytes()


def test_torch_peer_world1(eng):
    """The symmetric-memory fused path on a world of one: symmetric workspace,
    rendezvous, (empty) peer list and the stream barrier, against the golden run."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2603_03150_b200.sharded import run_pdhg_sharded

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        gm = load_golden("config0_s0")
        T = eng.types()
        try:
            pt, st = run_pdhg_sharded(gm, T.PdhgParams(eps_rel=1e-4), G=1, comm_kind="torch_peer")
        except (RuntimeError, NotImplementedError) as e:   # no symmetric memory on this stack
            pytest.skip(f"symmetric memory unavailable: {e}")
        r = gm.run("e4")
        assert st.status.value == "Optimal"
        assert st.iterations == int(r["iterations"]) and st.restarts == int(r["restarts"])
        # the fused path's periods (peer stores + device-side barriers) replay as graphs
        from paper_2603_03150_b200.engine import run_on_device
        from paper_2603_03150_b200.sharded import build_sharded

        dev = build_sharded(gm, 1, comm_kind="torch_peer")
        pt2, st2 = run_on_device(dev, gm, T.PdhgParams(eps_rel=1e-4))
        assert dev.graph and dev._graphs, "torch_peer periods were not captured"
        assert st2.iterations == st.iterations and pt2.x.tobytes() == pt.x.tobytes()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("kind", ["loopback", "loopback_fused"])
def test_failure_stops_every_shard(eng, G, kind):
    """Non-finite iterate on the last shard only (iteration 335, mid-period):
    every shard's fail word reads 335 (pdhg_set_peers which = 2) and the run
    returns the reference's failure exit."""
    from test_sharded_cpu import failing_block_model

    from paper_2603_03150_b200.engine import run_on_device
    from paper_2603_03150_b200.sharded import build_sharded

    p = failing_block_model()
    T = eng.types()
    params = T.PdhgParams(eps_rel=1e-6, max_kkt_passes=500)
    dev = build_sharded(p, G, comm_kind=kind)
    pt, st = run_on_device(dev, p, params)
    opt, ost = oracle.run_pdhg(p, oracle.PdhgParams(eps_rel=1e-6, max_kkt_passes=500))
    assert ost.status.value == "NumericalFailure" and ost.iterations == 335
    assert st.status.value == ost.status.value and st.iterations == ost.iterations
    assert [s.fail_iter() for s in dev.shards] == [335] * G
    np.testing.assert_allclose(pt.x, opt.x, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(pt.y, opt.y, rtol=1e-9, atol=1e-12)


def test_failure_single_gpu(eng):
    """The same failure exit on one GPU (the kernels' atomicMin fail word)."""
    from test_sharded_cpu import failing_block_model

    p = failing_block_model()
    T = eng.types()
    pt, st = eng.run_pdhg(p, T.PdhgParams(eps_rel=1e-6, max_kkt_passes=500))
    opt, ost = oracle.run_pdhg(p, oracle.PdhgParams(eps_rel=1e-6, max_kkt_passes=500))
    assert st.status.value == "NumericalFailure" and st.iterations == ost.iterations == 335
    np.testing.assert_allclose(pt.x, opt.x, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(pt.y, opt.y, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("kind", ["loopback", "loopback_fused"])
def test_sharded_sell_layouts_match_single_gpu(eng, kind):
    """Shards whose operators run on the sliced-ELL kernels (step, check,
    power iteration; 6 entries in flight for A', 4 for A) reproduce the
    single-GPU SELL run: same iterations, iterates to 1e-9."""
    from paper_2603_03150_b200.instances import config4
    from paper_2603_03150_b200.sharded import run_pdhg_sharded

    p = config4(scale=0.01, seed=21)
    T = eng.types()
    opts = eng.GpuOptions(sell="on", cache_layout=False)
    params = T.PdhgParams(eps_rel=1e-12, max_kkt_passes=256)
    p1, s1 = eng.run_pdhg(p, params, gpu=opts)
    p2, s2 = run_pdhg_sharded(p, params, G=2, gpu=opts, comm_kind=kind)
    assert s1.iterations == s2.iterations == 256 and s1.restarts == s2.restarts
    np.testing.assert_allclose(p2.x, p1.x, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(p2.y, p1.y, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("kind", ["loopback", "loopback_fused"])
def test_sharded_medium_rows_match_reference(eng, kind):
    """Shards with every longer-than-lanes row on the warp-per-row tier
    reproduce the golden run."""
    from paper_2603_03150_b200.sharded import run_pdhg_sharded

    gm = load_golden("config0_s0")
    T = eng.types()
    opts = eng.GpuOptions(sell="off", medium_per_lane=1)
    pt, st = run_pdhg_sharded(gm, T.PdhgParams(eps_rel=1e-4), G=2, gpu=opts, comm_kind=kind)
    r = gm.run("e4")
    assert st.status.value == "Optimal"
    assert st.iterations == int(r["iterations"]) and st.restarts == int(r["restarts"])
    assert float(gm.c @ pt.x) == pytest.approx(float(r["obj"]), rel=1e-6)


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("name", ["config0_s0", "eq_20x35_s17_ruiz"])
def test_overlap_is_bitwise_the_serial_split_schedule(eng, G, name):
    """The overlapped schedule (pass 0 of each split half step while the
    all-gather runs on a side stream) computes exactly what the same split
    kernels compute with the all-gather in line: bitwise-identical results."""
    from paper_2603_03150_b200.sharded import run_pdhg_sharded

    gm = load_golden(name)
    T = eng.types()
    params = T.PdhgParams(eps_rel=1e-4)
    pa, sa = run_pdhg_sharded(gm, params, G=G, gpu=eng.GpuOptions(), comm_kind="loopback", overlap="serial")
    pb, sb = run_pdhg_sharded(gm, params, G=G, gpu=eng.GpuOptions(), comm_kind="loopback", overlap="on")
    assert (sa.status, sa.iterations, sa.restarts) == (sb.status, sb.iterations, sb.restarts)
    assert pa.x.tobytes() == pb.x.tobytes() and pa.y.tobytes() == pb.y.tobytes()
    assert pa.z.tobytes() == pb.z.tobytes()


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("name,eps,limit", [("config0_s0", 1e-4, 200_000),
                                            ("ineq_12x20_s32_ruiz", 1e-4, 200_000),
                                            ("eq_10x18_s7_ruiz", 1e-12, 128)])
def test_overlap_matches_reference(eng, G, name, eps, limit):
    """Overlapped split schedule against the reference's golden runs."""
    from paper_2603_03150_b200.sharded import run_pdhg_sharded

    gm = load_golden(name)
    T = eng.types()
    pt, st = run_pdhg_sharded(gm, T.PdhgParams(eps_rel=eps, max_kkt_passes=limit), G=G,
                              gpu=eng.GpuOptions(), comm_kind="loopback", overlap="on")
    r = gm.run({1e-4: "e4", 1e-12: "lim128"}[eps])
    assert st.status.value == str(r["status"])
    assert st.iterations == int(r["iterations"])
    assert st.restarts == int(r["restarts"])
    scale = max(1.0, float(np.max(np.abs(r["x"]))))
    assert float(np.max(np.abs(pt.x - r["x"]))) <= 1e-9 * scale


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("name", ["config0_s0", "ineq_12x20_s32_ruiz"])
def test_overlap_sell_parts_match_csr_split(eng, G, name):
    """The split half steps over sliced-ELL parts (pass 0 = local-slot
    entries, pass 1 = the rest + epilogue, one fma chain per row) against the
    CSR-vector split kernels (sell="off"): same run to 1e-4, x to 1e-9."""
    from paper_2603_03150_b200.sharded import build_sharded, run_pdhg_sharded

    gm = load_golden(name)
    on = eng.GpuOptions(sell="on")
    dev = build_sharded(gm, G, comm_kind="loopback", overlap="on", opts=on)
    assert all(s._sell_part["A"] is not None and s._sell_part["At"] is not None for s in dev.shards)
    assert all(s._sell_part["A"] is None for s in
               build_sharded(gm, G, comm_kind="loopback", overlap="on",
                             opts=eng.GpuOptions(sell="off")).shards)
    T = eng.types()
    params = T.PdhgParams(eps_rel=1e-4)
    pa, sa = run_pdhg_sharded(gm, params, G=G, gpu=on, comm_kind="loopback", overlap="on")
    pb, sb = run_pdhg_sharded(gm, params, G=G, gpu=eng.GpuOptions(sell="off"), comm_kind="loopback",
                              overlap="on")
    assert (sa.status, sa.iterations, sa.restarts) == (sb.status, sb.iterations, sb.restarts)
    scale = max(1.0, float(np.max(np.abs(pb.x))))
    assert float(np.max(np.abs(pa.x - pb.x))) <= 1e-9 * scale


def test_overlap_config4_instance_matches_single_gpu(eng):
    """A 2M-nnz config-4 instance, 4 loopback shards, overlapped split
    schedule vs the single-GPU engine to 1e-4 (iterations within 5 %,
    objective 1e-6, the point passes the oracle's test), the serial split
    schedule bit for bit, and most entries in pass 0 (band-aligned shards)."""
    from paper_2603_03150_b200.instances import config4
    from paper_2603_03150_b200.sharded import ShardPlan, run_pdhg_sharded

    p = config4(scale=0.01, seed=21)
    T = eng.types()
    p1, s1 = eng.run_pdhg(p, T.PdhgParams(eps_rel=1e-4))
    p4, s4 = run_pdhg_sharded(p, T.PdhgParams(eps_rel=1e-4), G=4, comm_kind="loopback", overlap="on")
    assert s1.status.value == s4.status.value == "Optimal"
    assert abs(s4.iterations - s1.iterations) <= 0.05 * s1.iterations
    assert float(p.c @ p4.x) == pytest.approx(float(p.c @ p1.x), rel=1e-6)
    t = oracle.check_relative_termination(Model(p.A, p.b, p.c), KktPoint(p4.x, p4.y, p4.z), 1e-4)
    assert t.ok
    params = T.PdhgParams(eps_rel=1e-12, max_kkt_passes=256)
    pa, _ = run_pdhg_sharded(p, params, G=4, comm_kind="loopback", overlap="serial")
    pb, _ = run_pdhg_sharded(p, params, G=4, comm_kind="loopback", overlap="on")
    assert pa.x.tobytes() == pb.x.tobytes() and pa.y.tobytes() == pb.y.tobytes()
    # the same with both operators' split steps forced onto sliced-ELL parts
    # (heavy rows of A whole in pass 1)
    on = eng.GpuOptions(sell="on")
    pa, _ = run_pdhg_sharded(p, params, G=4, gpu=on, comm_kind="loopback", overlap="serial")
    pb, _ = run_pdhg_sharded(p, params, G=4, gpu=on, comm_kind="loopback", overlap="on")
    assert pa.x.tobytes() == pb.x.tobytes() and pa.y.tobytes() == pb.y.tobytes()
    plan = ShardPlan(p.A, 4)
    blk = plan.block(1, p.A, p.b, p.c, local_first=True)
    assert blk.a_nloc.sum() > 0.6 * blk.A.nnz and blk.at_nloc.sum() > 0.6 * blk.At.nnz


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("overlap", ["off", "on"])
def test_failure_replay_without_shared_fail_words(eng, G, overlap):
    """CUDA shards whose fail words are NOT connected (the NCCL all-gather
    mode's situation): the period with the non-finite iterate is replayed from
    its start up to iteration 335, so every shard stops there and the running
    averages equal the shared-fail-word run's bit for bit."""
    from test_sharded_cpu import failing_block_model

    from paper_2603_03150_b200.engine import DeviceLp, run_on_device
    from paper_2603_03150_b200.sharded import LoopbackComm, ShardedDevice, ShardPlan, build_sharded

    import torch

    p = failing_block_model()
    T = eng.types()
    params = T.PdhgParams(eps_rel=1e-6, max_kkt_passes=500)
    ref = build_sharded(p, G, comm_kind="loopback", overlap="serial" if overlap == "on" else "off")
    pr, sr = run_on_device(ref, p, params)
    plan = ShardPlan(p.A, G)
    stream = torch.cuda.Stream()
    split = overlap == "on"
    shards = [DeviceLp(b.A, b.b, b.c, eng.GpuOptions(), shard=b, stream=stream)
              for b in (plan.block(g, p.A, p.b, p.c, local_first=split) for g in range(G))]
    dev = ShardedDevice(plan, shards, LoopbackComm(plan), overlap=overlap)   # no connect_fail
    assert not dev._shared_fail()
    pt, st = run_on_device(dev, p, params)
    assert st.status.value == sr.status.value == "NumericalFailure"
    assert st.iterations == sr.iterations == 335
    assert pt.x.tobytes() == pr.x.tobytes() and pt.y.tobytes() == pr.y.tobytes()
    for a, b in zip(dev.shards, ref.shards):
        for nm in ("xbar", "ybar"):
            assert a.vec(nm).cpu().numpy().tobytes() == b.vec(nm).cpu().numpy().tobytes(), nm
