"""The consumer of the path: the reference IPM warm-started from the GPU PDHG point.

Two halves, because the GPU box has no /root/reference and this container
has no GPU:

    # on the GPU box: solve config 0 (the golden, reference-prepared model) to 1e-4 / 1e-6
    python tools/ipm_handoff.py gpu            -> gpurun_out/ipm_handoff_gpu.npz
    # here, with the reference importable: warm-start its IPM from those points
    python tools/ipm_handoff.py ref            -> profiles/r01_ipm_handoff.json

The ref half compares, for each tolerance, the reference IPM warm-started
from the GPU point with the same IPM warm-started from the reference's own
PDHG point (warmstart.py:99-154) and with the cold IPM (ipm.py:234), and
the IPM warm-started from the device's centered_start of the GPU point
(csrc/finish.cu k_center).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
OUT_GPU = ROOT / "gpurun_out" / "ipm_handoff_gpu.npz"
OUT_REF = ROOT / "profiles" / "r01_ipm_handoff.json"
EPS = (1e-4, 1e-6)


def gpu_half():
    import paper_2603_03150_b200 as eng
    from conftest import load_golden
    from paper_2603_03150_b200 import finish

    gm = load_golden("config0_s0")
    T = eng.types()
    d = {}
    for eps in EPS:
        pt, st = eng.run_pdhg(gm, T.PdhgParams(eps_rel=eps))
        tag = f"e{int(round(-np.log10(eps)))}"
        d[f"{tag}_x"], d[f"{tag}_y"], d[f"{tag}_z"] = pt.x, pt.y, pt.z
        d[f"{tag}_iterations"] = st.iterations
        d[f"{tag}_status"] = st.status.value
        cs = finish.centered_start(pt)   # the hand-off on the device (warmstart.py:99-107)
        d[f"{tag}_cs_x"], d[f"{tag}_cs_y"], d[f"{tag}_cs_z"] = cs.x, cs.y, cs.z
    OUT_GPU.parent.mkdir(exist_ok=True)
    np.savez(OUT_GPU, **d)
    print("wrote", OUT_GPU)


def ref_half():
    sys.path.insert(0, "/root/reference/pkg/src")
    import hybridlp
    from hybridlp import IpmParams, KktPoint, WarmStartParams, centered_start, run_ipm
    from hybridlp.warmstart import finish_point, prepare_model, warm_started_ipm

    from conftest import load_golden
    from paper_2603_03150_b200.instances import config0_general

    A, b, c, _, _ = config0_general(seed=0)
    g = hybridlp.GeneralLp(c=c, A=A, senses=[hybridlp.EQ] * A.shape[0], rhs=b,
                           lower=np.zeros(A.shape[1]), upper=np.full(A.shape[1], np.inf))
    prep = prepare_model(g)
    p = prep.solve_model
    gm = load_golden("config0_s0")
    assert np.array_equal(p.A.toarray(), gm.A.toarray()) and np.array_equal(p.b, gm.b)
    gpu = np.load(OUT_GPU)
    res = {"model": "config 0 (seed 0) after the reference prepare_model", "m": p.m, "n": p.n}
    _, cold = run_ipm(p, IpmParams())
    res["ipm_cold_iterations"] = cold.iterations
    for eps in EPS:
        tag = f"e{int(round(-np.log10(eps)))}"
        row = {"gpu_pdhg_iterations": int(gpu[f"{tag}_iterations"])}
        ref_pt, ref_st = hybridlp.run_pdhg(p, hybridlp.PdhgParams(eps_rel=eps))
        row["ref_pdhg_iterations"] = ref_st.iterations
        for who, pt in (("gpu", KktPoint(gpu[f"{tag}_x"], gpu[f"{tag}_y"], gpu[f"{tag}_z"])),
                        ("ref", ref_pt)):
            start = centered_start(pt, WarmStartParams())
            w = warm_started_ipm(p, start, IpmParams(), WarmStartParams())
            fin = finish_point(prep, w.point)
            row[f"{who}_warm_ipm_iterations"] = w.stats.iterations
            row[f"{who}_warm_ipm_status"] = w.stats.status.value
            row[f"{who}_final_max_violation"] = fin.violation.max_violation
        row["point_max_abs_diff_x"] = float(np.max(np.abs(gpu[f"{tag}_x"] - ref_pt.x)))
        if f"{tag}_cs_x" in gpu.files:   # device centered_start -> reference warm IPM
            ref_cs = centered_start(KktPoint(gpu[f"{tag}_x"], gpu[f"{tag}_y"], gpu[f"{tag}_z"]),
                                    WarmStartParams())
            dev_cs = KktPoint(gpu[f"{tag}_cs_x"], gpu[f"{tag}_cs_y"], gpu[f"{tag}_cs_z"])
            row["device_centered_start_max_rel_diff"] = float(max(
                np.max(np.abs(dev_cs.x - ref_cs.x) / np.maximum(np.abs(ref_cs.x), 1e-300)),
                np.max(np.abs(dev_cs.z - ref_cs.z) / np.maximum(np.abs(ref_cs.z), 1e-300))))
            w = warm_started_ipm(p, dev_cs, IpmParams(), WarmStartParams())
            fin = finish_point(prep, w.point)
            row["gpu_device_centered_warm_ipm_iterations"] = w.stats.iterations
            row["gpu_device_centered_final_max_violation"] = fin.violation.max_violation
        res[tag] = row
    OUT_REF.write_text(json.dumps(res, indent=1))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"gpu": gpu_half, "ref": ref_half}[sys.argv[1]]()
