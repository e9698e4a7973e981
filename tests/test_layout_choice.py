"""The automatic layout choices that decide which kernels a model runs (CPU:
the decisions are pure functions of the row-length profile)."""

from __future__ import annotations

import numpy as np
import torch

from paper_2603_03150_b200.engine import GpuOptions, _slice_pad, _want_row_order, auto_lanes, heavy_threshold
from paper_2603_03150_b200.instances import config2, config4


def _ptr(inst):
    return torch.from_numpy(np.asarray(inst.A.indptr, dtype=np.int64))


def test_config4_rows_are_renumbered_config2_rows_are_not():
    """Lognormal rows (config 4's A) get renumbered + sliced ELL; power-law
    rows (config 2's A: half the entries in rows over 4x the mean) stay on
    CSR-vector -- one lane per long row would serialise it."""
    opts = GpuOptions(sell_min_nnz=1)
    for inst, want in ((config4(scale=0.01, seed=4), True), (config2(scale=0.05, seed=2), False)):
        ptr = _ptr(inst)
        nnz, m = int(inst.A.nnz), inst.A.shape[0]
        H = heavy_threshold(auto_lanes(nnz, m))
        assert _want_row_order(torch, opts, ptr, nnz, H) is want, inst.name


def test_row_order_respects_options():
    inst = config4(scale=0.01, seed=4)
    ptr, nnz = _ptr(inst), int(inst.A.nnz)
    assert _want_row_order(torch, GpuOptions(), ptr, nnz, 512) is False       # below sell_min_nnz
    assert _want_row_order(torch, GpuOptions(row_order="length"), ptr, nnz, 512) is True
    assert _want_row_order(torch, GpuOptions(row_order="natural", sell_min_nnz=1), ptr, nnz, 512) is False
    assert _want_row_order(torch, GpuOptions(sell="off", sell_min_nnz=1), ptr, nnz, 512) is False


def test_slice_pad_of_sorted_rows_is_one():
    """Rows sorted by length inside windows pad to ~1.0; config 4's natural
    order pads ~4x (why the dual step needed the renumbering)."""
    inst = config4(scale=0.01, seed=4)
    lens = np.diff(inst.A.indptr)
    assert _slice_pad(torch, _ptr(inst), 512) > 3.0
    order = np.argsort(-lens, kind="stable")
    sorted_ptr = torch.from_numpy(np.concatenate([[0], np.cumsum(lens[order])]).astype(np.int64))
    assert _slice_pad(torch, sorted_ptr, 512) < 1.05


def test_length_order_long_first_windows():
    """_length_order (the row / column renumbering): a permutation; rows longer
    than `first` come first, window by window; inside each group and window
    by decreasing length, ties in the original order (stable)."""
    from paper_2603_03150_b200.engine import _length_order

    rng = np.random.default_rng(7)
    lens = torch.from_numpy(rng.integers(0, 80, 1000).astype(np.int64))
    W, first = 64, 32
    perm = _length_order(torch, "cpu", lens, W, first).numpy()
    L = lens.numpy()
    assert sorted(perm.tolist()) == list(range(1000))
    longs = L[perm] > first
    k = int(longs.sum())
    assert longs[:k].all() and not longs[k:].any()
    for part in (perm[:k], perm[k:]):
        win = part // W
        assert np.all(np.diff(win) >= 0)                       # window by window
        for w in np.unique(win):
            idx = part[win == w]
            lw = L[idx]
            assert np.all(np.diff(lw) <= 0)                     # longest first
            for v in np.unique(lw):                             # stable among ties
                same = idx[lw == v]
                assert np.all(np.diff(same) > 0)


def test_length_order_plain_windows_and_classes():
    from paper_2603_03150_b200.engine import _length_order

    lens = torch.tensor([3, 9, 1, 9, 5, 2, 40, 7], dtype=torch.int64)
    # plain windows of 4: [9, 9, 3, 1] then [40, 7, 5, 2]
    assert _length_order(torch, "cpu", lens, 4, 0).tolist() == [1, 3, 0, 2, 6, 7, 4, 5]
    # log2 classes, longest class first, one window: 40 | 9 9 | 5 7 | 3 2 | 1
    assert _length_order(torch, "cpu", lens, 8, -1).tolist() == [6, 1, 3, 7, 4, 0, 5, 2]
