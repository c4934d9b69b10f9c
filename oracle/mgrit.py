"""MGRIT-FAS engine restated for one worker, sweeps batched over C-intervals
(oracle).  Order of operations follows reference mgrit.py:

  _fc_sweep        mgrit.py:378-393      _restrict_sweep  mgrit.py:395-450
  _coarsest_solve  mgrit.py:452-495      _ascend          mgrit.py:497-571
  _probe/_measure  mgrit.py:573-598,754-761
  _vcycle/_fcycle  mgrit.py:602-635      _nested_iterations mgrit.py:659-675
  solve            mgrit.py:692-752      _materialize     mgrit.py:763-794

Every sweep of the reference starts from *pre-sweep* C-values (the start of
interval k is c_store[k-1] as it was before the sweep, mgrit.py:386), so the
F-offset j of all intervals is one batched Phi call here.  The problem must
offer step_batch(U[B, n], t_prev[B], t_next[B], spatial_level, smooth).
"""

import time
from dataclasses import dataclass, field

import numpy as np

from .fem2d import NewtonConvergenceError, joule_loss
from .spatial2d import assign_spatial_levels
from .state import BlockState, SpaceTimeVector

QOI_FLOOR = 1e-30


@dataclass(frozen=True)
class CycleSpec:
    kind: str = "V"
    gamma: int = 1
    max_iters: int = 50
    spatial_strategy: str = "none"
    nested_iterations: bool = False


@dataclass(frozen=True)
class StoppingCriterion:
    kind: str = "residual-norm"
    tolerance: float = 1e-8


@dataclass
class SolverRun:
    converged: bool = False
    iterations: int = 0
    residual_norms: list = field(default_factory=list)
    qoi_changes: list = field(default_factory=list)
    initial_residual: float = 0.0
    solve_seconds: float = 0.0
    failure: str = None
    phi_columns: int = 0


def qoi_change(p_new, p_old, floor=QOI_FLOOR):
    p_new = np.asarray(p_new, dtype=float)
    p_old = np.asarray(p_old, dtype=float)
    if p_new.size == 0:
        return 0.0
    return float(np.max(np.abs(p_new - p_old) / np.maximum(np.abs(p_old), floor)))


class _Level:
    def __init__(self, problem, index, grid, splitting, s_level):
        self.index = index
        self.t = grid.points
        self.n_points = grid.n_points
        self.m = splitting.factor
        self.c_idx = splitting.c_indices[1:]          # closing C-points
        self.K = len(self.c_idx)
        self.s = s_level
        # state rows are [field | scalars] (problems with n_scalars > 0, e.g.
        # the surrogate machine, problems.py:247-287)
        self.nf = problem.spatial.size(s_level)
        self.ns = int(getattr(problem, "n_scalars", 0))
        self.n = self.nf + self.ns
        self.anchor = np.zeros(self.n)
        self.c_store = np.zeros((self.K, self.n))
        self.u_keep = np.zeros((self.n_points, self.n)) if index > 0 else None
        self.rhs = np.zeros((self.n_points, self.n)) if index > 0 else None
        self.use_rhs = False

    def starts(self):
        """Pre-sweep start state of every interval: anchor, c_store[:-1]."""
        return np.vstack([self.anchor[None], self.c_store[:-1]])[:self.K]


class MgritOracle:
    def __init__(self, problem, hierarchy, cycle=None, stopping=None):
        self.problem = problem
        self.cycle = cycle or CycleSpec()
        self.stopping = stopping or StoppingCriterion()
        n_levels = hierarchy.n_levels
        if self.cycle.kind == "two-level" and n_levels > 2:
            n_levels = 2
        self.n_levels = n_levels
        self.assignment = assign_spatial_levels(
            self.cycle.spatial_strategy, n_levels, problem.spatial.n_grids)
        self.levels = [_Level(problem, l, hierarchy[l], hierarchy.splittings[l],
                              self.assignment[l]) for l in range(n_levels)]
        self.weights = problem.loss_weights(self.assignment[0])
        self.smooth = False
        self.phi_columns = 0

    # --- batched primitives ---
    def _phi(self, lvl, U, points, add_rhs=True):
        """U[b] advanced from t[points[b]-1] to t[points[b]], then the level
        rhs added (the `cur = step(); cur += rhs_at(i)` of mgrit.py:372-375)."""
        points = np.asarray(points)
        if not len(points):
            return np.zeros((0, lvl.n))
        self.phi_columns += len(points)
        out = self.problem.step_batch(U, lvl.t[points - 1], lvl.t[points],
                                      lvl.s, self.smooth)
        if add_rhs and lvl.use_rhs:
            out = out + lvl.rhs[points]
        return out

    def _walk(self, lvl, start):
        """F-walk of every interval; returns the last F-state per interval."""
        cur = start
        base = lvl.c_idx - lvl.m
        for j in range(1, lvl.m):
            cur = self._phi(lvl, cur, base + j)
        return cur

    def _R(self, fine, coarse, X):
        """restrict_state: field restricted, scalars copied (spatial.py:64-71)."""
        if coarse.s == fine.s:
            return X.copy()
        return np.stack([np.concatenate([self.problem.spatial.restrict_field(x[:fine.nf], fine.s),
                                         x[fine.nf:]]) for x in X])

    def _P(self, fine, coarse, X):
        """prolong_error: field interpolated, scalars copied (spatial.py:73-84)."""
        if coarse.s == fine.s:
            return X
        return np.stack([np.concatenate([self.problem.spatial.prolong_field(x[:coarse.nf], coarse.s),
                                         x[coarse.nf:]]) for x in X])

    # --- sweeps ---
    def _fc_sweep(self, lvl):
        last_f = self._walk(lvl, lvl.starts())
        lvl.c_store = self._phi(lvl, last_f, lvl.c_idx)

    def _restrict_sweep(self, lvl, nxt):
        starts = lvl.starts()
        last_f = self._walk(lvl, starts)
        prop = self._phi(lvl, last_f, lvl.c_idx, add_rhs=False)
        res = prop - lvl.c_store                       # mgrit.py:417-420
        if lvl.use_rhs:
            res = res + lvl.rhs[lvl.c_idx]
        kept = self._R(lvl, nxt, lvl.c_store)
        left_kept = self._R(lvl, nxt, starts)
        j = np.arange(1, lvl.K + 1)
        cprop = self._phi(nxt, left_kept, j, add_rhs=False)   # mgrit.py:424
        rhs = kept - cprop + self._R(lvl, nxt, res)
        nxt.u_keep[j] = kept
        nxt.rhs[j] = rhs
        nxt.use_rhs = True
        nxt.c_store = nxt.u_keep[nxt.c_idx].copy()

    def _coarsest_solve(self, lvl, nested=False):
        v = lvl.anchor.copy()
        vals = np.zeros((lvl.n_points, lvl.n))
        for i in range(1, lvl.n_points):
            v = self._phi(lvl, v[None], [i])[0]
            vals[i] = v
        if nested:
            lvl.u_keep[1:] = vals[1:]
            lvl.c_store = lvl.u_keep[lvl.c_idx].copy()
        else:
            lvl.u_keep[1:] = vals[1:] - lvl.u_keep[1:]
            lvl.c_store = lvl.c_store + lvl.u_keep[lvl.c_idx]

    def _apply(self, fine, coarse, points, payload, inject):
        ok = points <= fine.K
        points, payload = points[ok], payload[ok]
        if not len(points):
            return
        pay = self._P(fine, coarse, payload)
        if inject:
            fine.c_store[points - 1] = pay
        else:
            fine.c_store[points - 1] += pay

    def _ascend(self, coarse, fine, inject=False, solved=False):
        if solved:
            pts = np.arange(1, coarse.n_points)
            self._apply(fine, coarse, pts, coarse.u_keep[pts].copy(), inject)
            return
        cur = coarse.starts()
        base = coarse.c_idx - coarse.m
        for j in range(1, coarse.m + 1):
            pts = base + j
            cur = coarse.c_store.copy() if j == coarse.m else self._phi(coarse, cur, pts)
            pay = cur.copy() if inject else cur - coarse.u_keep[pts]
            self._apply(fine, coarse, pts, pay, inject)
        # F-tail beyond the last C-point (mgrit.py:529-530)
        last = int(coarse.c_idx[-1]) if coarse.K else 0
        v = coarse.c_store[-1] if coarse.K else coarse.anchor
        for i in range(last + 1, coarse.n_points):
            v = self._phi(coarse, v[None], [i])[0]
            pay = v.copy() if inject else v - coarse.u_keep[i]
            self._apply(fine, coarse, np.array([i]), pay[None], inject)

    def _probe(self, lvl):
        last_f = self._walk(lvl, lvl.starts())
        prop = self._phi(lvl, last_f, lvl.c_idx, add_rhs=False)
        res = prop - lvl.c_store                       # mgrit.py:587-591
        if lvl.use_rhs:
            res = res + lvl.rhs[lvl.c_idx]
        sum_sq = 0.0
        nf = lvl.nf
        for k in range(lvl.K):                         # norm_sq, state.py:74-75
            sum_sq += float(res[k, :nf] @ res[k, :nf]) + float(res[k, nf:] @ res[k, nf:])
        losses = np.zeros(lvl.K)
        for k, c in enumerate(lvl.c_idx):
            dt = float(lvl.t[c] - lvl.t[c - 1])
            losses[k] = joule_loss(BlockState(last_f[k, :nf]), BlockState(lvl.c_store[k, :nf]),
                                   dt, self.weights)
        return sum_sq, losses

    # --- cycles ---
    def _descend(self, l):
        for _ in range(self.cycle.gamma):
            self._fc_sweep(self.levels[l])
        self._restrict_sweep(self.levels[l], self.levels[l + 1])

    def _vcycle(self, l):
        if l == self.n_levels - 1:
            self._coarsest_solve(self.levels[l])
            return
        self._descend(l)
        self._vcycle(l + 1)
        self._ascend(self.levels[l + 1], self.levels[l],
                     solved=(l + 1 == self.n_levels - 1))

    def _fcycle(self, l):
        if l == self.n_levels - 1:
            self._coarsest_solve(self.levels[l])
            return
        self._descend(l)
        self._fcycle(l + 1)
        self._ascend(self.levels[l + 1], self.levels[l],
                     solved=(l + 1 == self.n_levels - 1))
        if l > 0:
            self._vcycle(l)

    def _single(self):
        lvl = self.levels[0]
        v = lvl.anchor.copy()
        for i in range(1, lvl.n_points):
            v = self._phi(lvl, v[None], [i])[0]
            if i in set(lvl.c_idx.tolist()):
                lvl.c_store[list(lvl.c_idx).index(i)] = v

    def _iterate_once(self):
        if self.n_levels == 1:
            self._single()
        elif self.cycle.kind == "F":
            self._fcycle(0)
        else:
            self._vcycle(0)

    def _nested(self):
        self.smooth = True
        try:
            bottom = self.levels[-1]
            bottom.use_rhs = False
            self._coarsest_solve(bottom, nested=True)
            for l in range(self.n_levels - 2, -1, -1):
                self._ascend(self.levels[l + 1], self.levels[l], inject=True,
                             solved=(l + 1 == self.n_levels - 1))
                if l > 0:
                    self.levels[l].use_rhs = False
                    self._vcycle(l)
        finally:
            self.smooth = False

    def solve(self, gather_solution=True, initial_guess=None):
        run = SolverRun()
        for lvl in self.levels:
            lvl.c_store[:] = lvl.anchor
            lvl.use_rhs = False
        if initial_guess is not None:
            lvl0 = self.levels[0]
            lvl0.c_store = np.stack([np.concatenate([initial_guess[c].field,
                                                     initial_guess[c].scalars])
                                     for c in lvl0.c_idx])
        elif self.cycle.nested_iterations and self.n_levels > 1:
            try:
                self._nested()
            except NewtonConvergenceError as e:
                run.failure = str(e)
        t0 = time.perf_counter()
        try:
            if run.failure is None:
                s, prev = self._probe(self.levels[0])
                run.initial_residual = s ** 0.5
                for it in range(1, self.cycle.max_iters + 1):
                    self._iterate_once()
                    s, losses = self._probe(self.levels[0])
                    norm = s ** 0.5
                    change = qoi_change(losses, prev) if losses.size else 0.0
                    prev = losses
                    run.iterations = it
                    run.residual_norms.append(norm)
                    run.qoi_changes.append(change)
                    if self.n_levels == 1:
                        run.converged = True
                        break
                    val = norm if self.stopping.kind == "residual-norm" else change
                    if val < self.stopping.tolerance:
                        run.converged = True
                        break
        except NewtonConvergenceError as e:
            run.failure = str(e)
        run.solve_seconds = time.perf_counter() - t0
        run.phi_columns = self.phi_columns
        sol = None
        if gather_solution and run.failure is None:
            sol = self.materialize()
        return run, sol

    def materialize(self):
        lvl = self.levels[0]
        out = np.zeros((lvl.n_points, lvl.n))
        out[0] = lvl.anchor
        cur = lvl.starts()
        base = lvl.c_idx - lvl.m
        for j in range(1, lvl.m):
            cur = self._phi(lvl, cur, base + j)
            out[base + j] = cur
        out[lvl.c_idx] = lvl.c_store
        last = int(lvl.c_idx[-1]) if lvl.K else 0
        v = out[last]
        for i in range(last + 1, lvl.n_points):
            v = self._phi(lvl, v[None], [i])[0]
            out[i] = v
        return out


def mgrit_solve(problem, hierarchy, cycle=None, stopping=None,
                gather_solution=True, initial_guess=None):
    return MgritOracle(problem, hierarchy, cycle, stopping).solve(
        gather_solution, initial_guess)
