"""numpy test double of one shard context (the C ABI's sharded semantics).

Mirrors libpdhg_b200's shard contract -- full padded vectors, rows owned
through slice offsets, primal/dual half steps with the skip-after-failure
rule, per-shard check partials, restart / best bookkeeping -- with the
reference's numpy operations.  Used with sharded.ShardedDevice and a gloo
TorchComm to test the multi-GPU host logic on CPU.  Test-only: the product
has no CPU path.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import torch

from paper_2603_03150_b200 import _native as N

X_SPACE = ("x", "xe", "xbar", "xbest", "zbest", "tn1", "tn2")


class NumpyShard:
    stream = None

    def __init__(self, blk):
        self.A = sp.csr_matrix(blk.A)
        self.At = sp.csr_matrix(blk.At)
        self.b, self.c = np.asarray(blk.b, float), np.asarray(blk.c, float)
        self.m, self.n = self.A.shape[0], self.At.shape[0]
        self.m_full, self.n_full = blk.m_full, blk.n_full
        self.y_off, self.x_off = blk.y_off, blk.x_off
        self.v = {k: np.zeros(self.n_full if k in X_SPACE else self.m_full)
                  for k in X_SPACE + ("y", "ybar", "ybest", "tm1")}
        self.v["scalars"] = np.zeros(64)
        self.params = None
        self.fail = -1
        self.fail_peers = []
        # local_first blocks (split steps): each row's first nloc entries are the
        # shard's own slots -- pass 0 sums them, pass 1 the rest + epilogue
        self.split = {}
        for key, M, nloc in (("A", self.A, getattr(blk, "a_nloc", None)),
                             ("At", self.At, getattr(blk, "at_nloc", None))):
            if nloc is not None:
                pos = np.arange(M.nnz) - np.repeat(M.indptr[:-1], np.diff(M.indptr))
                first = pos < np.repeat(np.asarray(nloc), np.diff(M.indptr))
                rid = np.repeat(np.arange(M.shape[0]), np.diff(M.indptr))

                def part(mask, M=M, rid=rid):
                    ptr = np.concatenate([[0], np.cumsum(np.bincount(rid[mask], minlength=M.shape[0]))])
                    return sp.csr_matrix((M.data[mask], M.indices[mask], ptr), shape=M.shape)

                self.split[key] = (part(first), part(~first))
        self.partial = {}

    def vec(self, name):
        return torch.from_numpy(self.v[name])

    def _xs(self):
        return slice(self.x_off, self.x_off + self.n)

    def _ys(self):
        return slice(self.y_off, self.y_off + self.m)

    def reset(self):
        for k in ("x", "xe", "xbar", "y", "ybar"):
            self.v[k][:] = 0.0

    def set_step(self, iter0, tau_w, sigma_w, w0):
        self.params = (int(iter0), tau_w, sigma_w, w0)
        self.fail = -1

    def half_step_pass(self, primal, j, pass_):
        """Split half step (pdhg_half_step_pass): pass 0 = local-slot entries,
        pass 1 = the rest, added to the pass-0 partial, + the epilogue."""
        key = "At" if primal else "A"
        if key not in self.split:
            if pass_ == 0:
                self.half_step(primal, j)
            return
        loc, rem = self.split[key]
        v = self.v["y"] if primal else self.v["xe"]
        if pass_ == 0:
            self.partial[key] = loc @ v
            return
        self.half_step(primal, j, dot=self.partial.pop(key) + rem @ v)

    def half_step(self, primal, j, dot=None):
        iter0, tau_w, sigma_w, w0 = self.params
        it = iter0 + j + 1
        if self.fail >= 0 and self.fail < it:
            return
        w = w0 + (j + 1)
        if primal:
            xs = self._xs()
            x = self.v["x"][xs].copy()
            aty = self.At @ self.v["y"] if dot is None else dot
            xn = np.maximum(0.0, x - tau_w * (self.c - aty))
            self.v["x"][xs] = xn
            self.v["xe"][xs] = 2.0 * xn - x
            self.v["xbar"][xs] += (xn - self.v["xbar"][xs]) / w
            bad = not np.all(np.isfinite(xn))
        else:
            ys = self._ys()
            ax = self.A @ self.v["xe"] if dot is None else dot
            yn = self.v["y"][ys] + sigma_w * (self.b - ax)
            self.v["y"][ys] = yn
            self.v["ybar"][ys] += (yn - self.v["ybar"][ys]) / w
            bad = not np.all(np.isfinite(yn))
        if bad:
            for sh in [self] + self.fail_peers:   # pdhg_set_peers(which = 2)
                if sh.fail < 0 or it < sh.fail:
                    sh.fail = it

    def connect_fail(self, others):
        self.fail_peers = list(others)

    def fail_iter(self):
        return self.fail

    def _xy(self, spec):
        which = spec & 3
        if which == N.PT_AVG:
            return self.v["xbar"], self.v["ybar"]
        if which == N.PT_BEST:
            return self.v["xbest"], self.v["ybest"]
        return self.v["x"], self.v["y"]

    def check_device(self, *specs):
        out = self.v["scalars"]
        out[:] = 0.0
        xs, ys = self._xs(), self._ys()
        for k, spec in enumerate(specs):
            x, y = self._xy(spec)
            t = self.c - self.At @ y
            z = self.v["zbest"][xs] if spec & N.SPEC_BEST_Z else np.maximum(0.0, t)
            r_p = self.b - self.A @ x
            r_d = t - z
            q = out[k * N.NQ:(k + 1) * N.NQ]
            q[N.Q_RP2] = r_p.dot(r_p)
            q[N.Q_RPMAX] = np.max(np.abs(r_p)) if r_p.size else 0.0
            q[N.Q_BY] = float(self.b @ y[ys])
            q[N.Q_RD2] = r_d.dot(r_d)
            q[N.Q_RDMAX] = np.max(np.abs(r_d)) if r_d.size else 0.0
            q[N.Q_CX] = float(self.c @ x[xs])
            q[N.Q_XZ] = float(x[xs] @ z)
        return torch.from_numpy(out[:len(specs) * N.NQ])

    def restart(self, which):
        if which == N.PT_CUR:
            self.v["xbar"][:] = self.v["x"]
            self.v["ybar"][:] = self.v["y"]
        else:
            self.v["x"][:] = self.v["xbar"]
            self.v["y"][:] = self.v["ybar"]

    def reduced_costs(self, spec, out_name):
        x, y = self._xy(spec)
        self.v[out_name][self._xs()] = np.maximum(0.0, self.c - self.At @ y)

    def save_best(self, which, flags):
        x, y = self._xy(which)
        if flags & N.BEST_Z:
            self.reduced_costs(which, "zbest")
        if flags & N.BEST_XY and (which & 3) != N.PT_BEST:
            self.v["xbest"][:] = x
            self.v["ybest"][:] = y

    def spmv_named(self, transpose, in_name, out_name):
        if transpose:
            self.v[out_name][self._xs()] = self.At @ self.v[in_name]
        else:
            self.v[out_name][self._ys()] = self.A @ self.v[in_name]

    def sumsq_named(self, name):
        v = self.v[name][self._xs()]
        self.v["scalars"][0] = v.dot(v)
        return torch.from_numpy(self.v["scalars"][:1])

    def div_named(self, src, dst, s):
        xs = self._xs()
        self.v[dst][xs] = self.v[src][xs] / s
