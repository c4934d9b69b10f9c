"""CPU test double of GpuFemProblem's batched interface (tests only).

Lets the multi-rank orchestration of paper_1912_03106_b200.mgrit run under
torch.distributed/gloo on CPU.  Phi is the oracle's banded-Cholesky step
(oracle/fem2d.py), transfers are the oracle's; nothing here ships."""

import numpy as np
import torch
from scipy.linalg import cho_solve_banded, cholesky_banded

from oracle import fem2d


class CpuDoubleProblem:
    n_scalars = 0

    def __init__(self, spec):
        self.spec = spec
        self.oracle = fem2d.make_problem(spec)
        self.spatial = self.oracle.spatial
        self.device = torch.device("cpu")
        self.phases = self.oracle.levels[0].phases
        self.n_src = len(self.phases)
        self._fac = {}

    def source_values(self, times, smooth=False):
        times = np.atleast_1d(np.asarray(times, dtype=float))
        return np.stack([self.oracle.source_values(float(t), smooth) for t in times]) \
            if len(times) else np.zeros((0, self.n_src))

    def loss_weights(self, level=0):
        return torch.as_tensor(self.oracle.levels[level].lumped)

    def phi_batch(self, level, U, inv_dt, src, out, g=None, g_idx=None, guess=None):
        lv = self.oracle.levels[level]
        Un = U.numpy()
        MU = (lv.M @ Un.T).T
        F = src.numpy() @ lv.shapes
        for b, c in enumerate(inv_dt.numpy()):
            key = (level, float(c))
            if key not in self._fac:
                self._fac[key] = cholesky_banded(lv.to_banded(lv.K + lv.M * float(c)))
            x = cho_solve_banded((self._fac[key], False), F[b] + c * MU[b])
            if g is not None and int(g_idx[b]) >= 0:
                x = x + g[int(g_idx[b])].numpy()
            out[b] = torch.as_tensor(x)

    def restrict(self, fine, X, out):
        for b in range(X.shape[0]):
            out[b] = torch.as_tensor(self.spatial.restrict_field(X[b].numpy(), fine))

    def prolong_add(self, coarse, X, out, out_idx=None, beta=1.0):
        for b in range(X.shape[0]):
            o = int(out_idx[b]) if out_idx is not None else b
            v = torch.as_tensor(self.spatial.prolong_field(X[b].numpy(), coarse))
            out[o] = v if beta == 0.0 else out[o] + v

    def c_residual(self, level, prop, c, sumsq, c_idx=None, g=None, g_idx=None, res=None,
                   last_f=None, inv_dt=None, loss=None):
        w = self.loss_weights(level)
        for b in range(prop.shape[0]):
            cb = c[int(c_idx[b]) if c_idx is not None else b]
            r = prop[b] - cb
            if g is not None and (g_idx is None or int(g_idx[b]) >= 0):
                r = r + g[int(g_idx[b]) if g_idx is not None else b]
            if res is not None:
                res[b] = r
            sumsq[b] = torch.dot(r, r)
            if last_f is not None:
                du = (cb - last_f[b]) * inv_dt[b]
                loss[b] = torch.dot(w, du * du)

    def rows_axpby(self, B, out, a, c=None, sign=1, out_rows=None, a_rows=None, c_rows=None):
        def row(t, r, b):
            t2 = t if t.dim() == 2 else t.view(1, -1)
            if r is None:
                return t2[b]
            if isinstance(r, tuple):
                return t2[r[0] + b * r[1]]
            return t2[int(r[b])]
        for b in range(B):
            v = row(a, a_rows, b).clone()
            if c is not None:
                v = v + row(c, c_rows, b) if sign > 0 else v - row(c, c_rows, b)
            row(out, out_rows, b).copy_(v)

    def fas_rhs(self, coarse, coarsen, kept, cprop, res, out):
        for b in range(kept.shape[0]):
            rr = (torch.as_tensor(self.spatial.restrict_field(res[b].numpy(), coarse - 1))
                  if coarsen else res[b])
            out[b] = (kept[b] - cprop[b]) + rr
