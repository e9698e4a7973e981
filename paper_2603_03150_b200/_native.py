"""ctypes binding of libpdhg_b200.so (declared in include/pdhg_b200.h).

There is no fallback: if the library is missing or fails to load, every
entry point raises.  The product path has exactly one implementation, the
sm_100a kernels behind this ABI.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

# the product build; PDHG_B200_LIB points at another build of the same ABI
# (e.g. the experiment build: python -m paper_2603_03150_b200.build --experimental)
LIB_PATH = Path(os.environ.get("PDHG_B200_LIB") or Path(__file__).resolve().parent / "libpdhg_b200.so")

PT_CUR, PT_AVG, PT_BEST = 0, 1, 2
SPEC_BEST_Z = 16
BEST_XY, BEST_Z = 1, 2
NQ = 8
Q_RP2, Q_RPMAX, Q_BY, Q_RD2, Q_RDMAX, Q_CX, Q_XZ = range(7)

# every symbol include/pdhg_b200.h declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "pdhg_abi_version", "pdhg_last_error", "pdhg_workspace_bytes", "pdhg_ctx_create",
    "pdhg_ctx_destroy", "pdhg_spmv", "pdhg_opnorm", "pdhg_reset", "pdhg_run_period",
    "pdhg_check", "pdhg_restart", "pdhg_save_best", "pdhg_fetch", "pdhg_point_device", "pdhg_time_kernel",
    "pdhg_transpose_tmp_bytes", "pdhg_transpose_csr",
    "pdhg_psr_tmp_bytes", "pdhg_psr_plan", "pdhg_psr_build",
    "pdhg_check_device", "pdhg_vector", "pdhg_reduced_costs", "pdhg_set_step", "pdhg_half_step",
    "pdhg_fail_iter", "pdhg_sumsq", "pdhg_div", "pdhg_ruiz_tmp_bytes", "pdhg_ruiz",
    "pdhg_split_build", "pdhg_stdform_tmp_bytes", "pdhg_stdform_plan", "pdhg_stdform_build",
    "pdhg_spmv_seq", "pdhg_unscale_point", "pdhg_restrict_x", "pdhg_lift_x", "pdhg_lift_slacks",
    "pdhg_lift_bound_duals", "pdhg_max0", "pdhg_violation_tmp_bytes", "pdhg_violation",
    "pdhg_sell_tmp_bytes", "pdhg_sell_plan", "pdhg_sell_fill", "pdhg_sell_sort", "pdhg_set_peers",
    "pdhg_run_period_check", "pdhg_center_toward_target", "pdhg_dot_tmp_bytes", "pdhg_dot",
    "pdhg_permute_rows", "pdhg_features", "pdhg_half_step_pass", "pdhg_debug_oob",
    "pdhg_check_dot_enable", "pdhg_use_check_dot", "pdhg_check_fuse_enable",
)

VEC = {name: i for i, name in enumerate(
    ("x", "xe", "xbar", "xbest", "zbest", "tn1", "tn2", "y", "ybar", "ybest", "tm1", "scalars",
     "failword"))}


class Psr(C.Structure):
    """struct pdhg_psr (panel-staged rows layout of one operator)."""

    _fields_ = [
        ("rows", C.c_int32), ("cols", C.c_int32), ("R", C.c_int32), ("W", C.c_int32),
        ("nblk", C.c_int32), ("ntiles", C.c_int32), ("ngroups", C.c_int32), ("nent", C.c_int64),
        ("blk_tile_ptr", C.c_void_p), ("tile_bin", C.c_void_p), ("gstart", C.c_void_p),
        ("rcnt", C.c_void_p), ("val", C.c_void_p), ("col16", C.c_void_p), ("col", C.c_void_p),
        ("heavy", C.c_void_p),
    ]


class Sell(C.Structure):
    """struct pdhg_sell (sliced-ELL layout of one operator)."""

    _fields_ = [("rows", C.c_int32), ("nslices", C.c_int32), ("sptr", C.c_void_p),
                ("width", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p),
                ("perm", C.c_void_p), ("nslots", C.c_int64)]


class Problem(C.Structure):
    """struct pdhg_problem."""

    _fields_ = [
        ("m", C.c_int32), ("n", C.c_int32), ("nnz", C.c_int64),
        ("a_ptr", C.c_void_p), ("a_col", C.c_void_p), ("a_val", C.c_void_p),
        ("at_ptr", C.c_void_p), ("at_col", C.c_void_p), ("at_val", C.c_void_p),
        ("b", C.c_void_p), ("c", C.c_void_p),
        ("a_lanes", C.c_int32), ("at_lanes", C.c_int32), ("heavy_threshold", C.c_int32),
        ("a_n_heavy", C.c_int32), ("at_n_heavy", C.c_int32),
        ("a_heavy", C.c_void_p), ("at_heavy", C.c_void_p),
        ("a_psr", C.POINTER(Psr)), ("at_psr", C.POINTER(Psr)),
        ("l2_persist", C.c_int32),
        ("m_full", C.c_int32), ("n_full", C.c_int32), ("y_off", C.c_int32), ("x_off", C.c_int32),
        ("at_nnz", C.c_int64),
        ("a_nsplit", C.c_int32), ("a_split", C.c_void_p),
        ("at_heavy_threshold", C.c_int32),
        ("a_sell", C.POINTER(Sell)), ("at_sell", C.POINTER(Sell)),
        ("persistent", C.c_int32),
        ("a_light_max", C.c_int32), ("at_light_max", C.c_int32),
        ("a_n_medium", C.c_int32), ("at_n_medium", C.c_int32),
        ("a_medium", C.c_void_p), ("at_medium", C.c_void_p),
        ("at_nsplit", C.c_int32), ("at_split", C.c_void_p),
        ("a_sell_part", C.c_void_p * 2), ("a_part_ptr", C.c_void_p * 2),
        ("at_sell_part", C.c_void_p * 2), ("at_part_ptr", C.c_void_p * 2),
    ]


class NativeError(RuntimeError):
    pass


_lib = None
_lock = threading.Lock()


def _sig(lib, name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)


ABI_VERSION = 6   # include/pdhg_b200.h PDHG_ABI_VERSION


def load():
    """Load (once) and type the native library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeError(
                f"{LIB_PATH} not found: build it with `python -m paper_2603_03150_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        vp, i32, i64, dbl, szt = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_size_t
        P = C.POINTER
        _sig(lib, "pdhg_abi_version", C.c_int)
        _sig(lib, "pdhg_last_error", C.c_char_p)
        _sig(lib, "pdhg_workspace_bytes", szt, i32, i32)
        _sig(lib, "pdhg_ctx_create", C.c_int, P(Problem), vp, szt, vp, P(vp))
        _sig(lib, "pdhg_ctx_destroy", C.c_int, vp)
        _sig(lib, "pdhg_spmv", C.c_int, vp, C.c_int, vp, vp)
        _sig(lib, "pdhg_opnorm", C.c_int, vp, vp, dbl, i32, P(dbl), P(i32))
        _sig(lib, "pdhg_reset", C.c_int, vp)
        _sig(lib, "pdhg_run_period", C.c_int, vp, i32, i64, dbl, dbl, dbl, P(i64))
        _sig(lib, "pdhg_check", C.c_int, vp, i32, P(i32), P(dbl))
        _sig(lib, "pdhg_restart", C.c_int, vp, i32)
        _sig(lib, "pdhg_save_best", C.c_int, vp, i32, i32)
        _sig(lib, "pdhg_fetch", C.c_int, vp, i32, vp, vp, vp)
        _sig(lib, "pdhg_point_device", C.c_int, vp, i32, vp, vp, vp)
        _sig(lib, "pdhg_time_kernel", C.c_int, vp, i32, i32, dbl, dbl, P(dbl))
        _sig(lib, "pdhg_transpose_tmp_bytes", szt, i64, i32, i32)
        _sig(lib, "pdhg_transpose_csr", C.c_int, i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, szt, vp)
        _sig(lib, "pdhg_psr_tmp_bytes", szt, i32, i32, i64)
        _sig(lib, "pdhg_psr_plan", C.c_int, i32, i32, i64, vp, vp, i32, i32, vp, szt, vp,
             P(i32), P(i32), P(i32), P(i32), P(i32), P(i64), P(i64))
        _sig(lib, "pdhg_psr_build", C.c_int, i32, i32, i64, vp, vp, vp, i32, vp, szt, vp,
             vp, vp, vp, vp, vp, vp, vp, vp)
        _sig(lib, "pdhg_check_device", C.c_int, vp, i32, P(i32))
        _sig(lib, "pdhg_vector", vp, vp, i32)
        _sig(lib, "pdhg_reduced_costs", C.c_int, vp, i32, vp)
        _sig(lib, "pdhg_set_step", C.c_int, vp, i64, dbl, dbl, dbl)
        _sig(lib, "pdhg_half_step", C.c_int, vp, i32, i32)
        _sig(lib, "pdhg_fail_iter", C.c_int, vp, P(i64))
        _sig(lib, "pdhg_sumsq", C.c_int, vp, vp, i64, vp)
        _sig(lib, "pdhg_div", C.c_int, vp, vp, vp, i64, dbl)
        _sig(lib, "pdhg_ruiz_tmp_bytes", szt, i32, i32)
        _sig(lib, "pdhg_ruiz", C.c_int, i32, i32, i64, vp, vp, vp, vp, vp, i32, dbl, dbl, vp, szt, vp,
             P(i32))
        _sig(lib, "pdhg_split_build", C.c_int, i32, vp, vp, i32, i32, vp, vp, vp, P(i32))
        _sig(lib, "pdhg_stdform_tmp_bytes", szt, i32, i32)
        _sig(lib, "pdhg_stdform_plan", C.c_int, i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, szt, vp, vp)
        _sig(lib, "pdhg_stdform_build", C.c_int, i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp,
             vp, szt, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp)
        _sig(lib, "pdhg_spmv_seq", C.c_int, i32, vp, vp, vp, vp, vp, vp, vp)
        _sig(lib, "pdhg_unscale_point", C.c_int, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp)
        _sig(lib, "pdhg_restrict_x", C.c_int, i32, vp, vp, vp, vp, vp, vp)
        _sig(lib, "pdhg_lift_x", C.c_int, i32, vp, vp, vp, vp, vp, vp)
        _sig(lib, "pdhg_lift_slacks", C.c_int, i32, vp, vp, vp, vp, vp)
        _sig(lib, "pdhg_lift_bound_duals", C.c_int, i32, vp, vp, vp, vp)
        _sig(lib, "pdhg_max0", C.c_int, i64, vp, vp, vp)
        _sig(lib, "pdhg_violation_tmp_bytes", szt, i32, i32)
        _sig(lib, "pdhg_sell_tmp_bytes", szt, i32)
        _sig(lib, "pdhg_set_peers", C.c_int, vp, i32, vp, i32)
        _sig(lib, "pdhg_center_toward_target", C.c_int, i64, vp, vp, dbl, dbl, dbl, vp, vp, vp)
        _sig(lib, "pdhg_dot_tmp_bytes", szt)
        _sig(lib, "pdhg_dot", C.c_int, i64, vp, vp, vp, szt, vp, P(dbl))
        _sig(lib, "pdhg_run_period_check", C.c_int, vp, i32, i64, dbl, dbl, dbl, i32, P(i32), P(i64),
             P(dbl))
        _sig(lib, "pdhg_sell_plan", C.c_int, i32, vp, i32, vp, vp, vp, szt, vp, P(i64))
        _sig(lib, "pdhg_sell_sort", C.c_int, i32, vp, i32, vp, vp, vp)
        _sig(lib, "pdhg_sell_fill", C.c_int, i32, vp, vp, vp, i32, vp, vp, vp, vp, vp)
        _sig(lib, "pdhg_permute_rows", C.c_int, i32, vp, vp, vp, vp, vp, vp, vp, vp)
        _sig(lib, "pdhg_features", C.c_int)
        _sig(lib, "pdhg_check_dot_enable", C.c_int, vp, i32)
        _sig(lib, "pdhg_use_check_dot", C.c_int, vp, i32)
        _sig(lib, "pdhg_check_fuse_enable", C.c_int, vp, i32)
        _sig(lib, "pdhg_half_step_pass", C.c_int, vp, i32, i32, i32)
        _sig(lib, "pdhg_debug_oob", C.c_int, P(i64), P(i64), P(i64))
        _sig(lib, "pdhg_violation", C.c_int, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
             vp, szt, vp, P(dbl))
        if lib.pdhg_abi_version() != ABI_VERSION:
            raise NativeError("libpdhg_b200.so ABI version mismatch")
        _lib = lib
        return lib


FEATURE_EXPERIMENTAL = 1
FEATURE_BOUNDS_CHECK = 2


def bounds_checked() -> bool:
    return bool(load().pdhg_features() & FEATURE_BOUNDS_CHECK)


def debug_oob() -> tuple[int, int, int]:
    """(count, first index, its bound) of out-of-bounds loads since the last call
    (bounds-checked build only; resets the count)."""
    n, i, b = C.c_int64(), C.c_int64(), C.c_int64()
    check(load().pdhg_debug_oob(C.byref(n), C.byref(i), C.byref(b)))
    return int(n.value), int(i.value), int(b.value)


def experimental() -> bool:
    """True when the loaded library is the experiment build (PSR, persistent
    periods, L2 windows; measured slower, not in the product build)."""
    return bool(load().pdhg_features() & FEATURE_EXPERIMENTAL)


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.pdhg_last_error().decode(errors="replace") if _lib is not None else "?"
        raise NativeError(f"libpdhg_b200 error {rc}: {msg}")
