"""GPU-resident MGRIT-FAS engine with batched Phi.

Mirrors the order of operations of the reference MgritSolver
(mgrit.py:290-801) -- same sweeps, same FAS right-hand side, same coarsest
gather / sequential solve / scatter, same residual probe and stopping rule --
with one structural change: every sweep starts from *pre-sweep* C-values
(mgrit.py:381-392, :345-346), so F-offset j of all owned intervals is ONE
batched Phi call (pg_phi_batch over [K][n] device states) instead of K
sequential calls.  Everything lives in HBM: per level the C-store [K][n],
and on coarse levels the kept iterate and FAS right-hand side [n_owned][n]
(the lean layout of mgrit.py:14-24).

Multi-GPU: ranks own contiguous C-intervals per level (runtime.Decomposition,
= reference runtime.py:31-105); the left-boundary C-state is exchanged with
one grouped NCCL send/recv per sweep (mgrit.py:339-350), coarse-point
redistribution and the coarsest gather/scatter are grouped p2p
(mgrit.py:434-449, :458-480, :549-559), norms are rank-ordered sums.
"""

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import NewtonConvergenceError
from .runtime import Decomposition, NullTransport, plan_moves
from .spatial import assign_spatial_levels

CYCLE_KINDS = ("two-level", "V", "F")
STOPPING_KINDS = ("residual-norm", "qoi-change")
QOI_FLOOR = 1e-30


@dataclass(frozen=True)
class CycleSpec:
    """reference mgrit.py:49-64"""
    kind: str = "V"
    gamma: int = 1
    max_iters: int = 50
    spatial_strategy: str = "none"
    nested_iterations: bool = False

    def __post_init__(self):
        if self.kind not in CYCLE_KINDS:
            raise ValueError(f"cycle kind must be one of {CYCLE_KINDS}, got {self.kind!r}")
        if self.gamma < 0:
            raise ValueError(f"gamma must be >= 0, got {self.gamma}")
        if self.max_iters < 1:
            raise ValueError(f"max_iters must be >= 1, got {self.max_iters}")


@dataclass(frozen=True)
class StoppingCriterion:
    """reference mgrit.py:67-78"""
    kind: str = "residual-norm"
    tolerance: float = 1e-8

    def __post_init__(self):
        if self.kind not in STOPPING_KINDS:
            raise ValueError(f"stopping kind must be one of {STOPPING_KINDS}, "
                             f"got {self.kind!r}")
        if self.tolerance <= 0.0:
            raise ValueError(f"tolerance must be positive, got {self.tolerance}")


def qoi_change(p_new, p_old, floor=QOI_FLOOR):
    """reference mgrit.py:81-90"""
    p_new = np.asarray(p_new, dtype=float)
    p_old = np.asarray(p_old, dtype=float)
    if p_new.shape != p_old.shape:
        raise ValueError(f"sample shapes differ: {p_new.shape} vs {p_old.shape}")
    if p_new.size == 0:
        return 0.0
    return float(np.max(np.abs(p_new - p_old) / np.maximum(np.abs(p_old), floor)))


def storage_estimate(n_levels, n_fine_steps, factors, n_workers, sizes=None,
                     coarsest_factor=None):
    """reference mgrit.py:93-124"""
    factors = list(factors)
    if len(factors) != n_levels - 1:
        raise ValueError(f"{n_levels} levels need {n_levels - 1} factors, got {len(factors)}")
    if sizes is None:
        sizes = [1] * n_levels
    if len(sizes) != n_levels:
        raise ValueError(f"need one size per level, got {len(sizes)}")
    if coarsest_factor is None:
        coarsest_factor = factors[-1] if factors else 2
    prods = [1]
    for m in factors:
        prods.append(prods[-1] * m)
    prods.append(prods[-1] * coarsest_factor)
    total = 0
    for l in range(n_levels):
        total += math.ceil(n_fine_steps / (prods[l + 1] * n_workers)) * sizes[l]
        if l >= 1:
            total += 2 * math.ceil(n_fine_steps / (prods[l] * n_workers)) * sizes[l]
    return total


@dataclass
class StorageReport:
    per_level: list
    total: int
    estimate: int


@dataclass
class SolverRun:
    """reference mgrit.py:134-151, plus device statistics."""
    converged: bool = False
    iterations: int = 0
    residual_norms: list = field(default_factory=list)
    qoi_changes: list = field(default_factory=list)
    iteration_seconds: list = field(default_factory=list)
    initial_residual: float = 0.0
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0
    level_seconds: list = field(default_factory=list)
    storage: StorageReport = None
    n_workers: int = 1
    failure: str = None
    phi_columns: int = 0           # Phi applications (columns) on this rank
    phi_calls: int = 0             # batched Phi calls on this rank

    @property
    def total_seconds(self):
        return self.setup_seconds + self.solve_seconds


class _Boundary:
    """Left-boundary state of a sweep whose exchange may still be in flight."""

    __slots__ = ("buf", "pending")

    def __init__(self, buf, pending):
        self.buf, self.pending = buf, pending

    def ready(self):
        if self.pending is not None:
            self.pending.wait()
            self.pending = None
        return self.buf


def _drain(boundary):
    if boundary is not None:
        boundary.ready()


class _Level:
    """Per-rank device workspace of one time level."""

    def __init__(self, solver, index, grid, splitting, s_level):
        prob, T = solver.problem, solver.transport
        dev = prob.device
        f64 = dict(dtype=torch.float64, device=dev)
        self.index = index
        self.grid = grid
        self.t = grid.points
        self.n_points = grid.n_points
        self.splitting = splitting
        self.m = splitting.factor
        self.s = s_level
        # one state row = [field | scalars] (prob.state_size)
        self.n = prob.state_size(s_level) if hasattr(prob, "state_size") \
            else prob.spatial.size(s_level)
        self.decomp = d = Decomposition(splitting, T.size)
        r = T.rank
        self.empty = d.is_empty(r)
        self.K = 0 if self.empty else d.n_units(r)
        self.first = d.first_unit(r)
        self.c_idx = np.asarray(d.c_points(r), dtype=np.int64) if not self.empty \
            else np.zeros(0, np.int64)
        self.own_lo, self.own_hi = d.owned_range(r)
        self.left_index = d.left_boundary_index(r) if not self.empty else 0
        self.n_owned = max(self.own_hi - self.own_lo, 0)
        self.anchor = torch.zeros(self.n, **f64)
        self.c_store = torch.zeros(self.K, self.n, **f64)
        self.u_keep = self.rhs = None
        if index > 0:
            self.u_keep = torch.zeros(self.n_owned, self.n, **f64)
            self.rhs = torch.zeros(self.n_owned, self.n, **f64)
        self.use_rhs = False
        self.seconds = 0.0
        self.chain_vals = None          # coarsest chain values (rank 0)
        self.full_rhs = None            # gathered coarsest rhs (rank 0, multi-rank)
        self.chain_graphs = {}          # captured coarsest chains
        # per-point tables (device): 1/dt and source values at t_next
        t = self.t
        inv = np.zeros(self.n_points)
        inv[1:] = 1.0 / (t[1:] - t[:-1])                 # dt = t_next - t_prev
        self.inv_dt_all = torch.as_tensor(inv, **f64)
        self.inv_dt_all_h = inv
        src = [prob.source_values(t, smooth=False), prob.source_values(t, smooth=True)]
        self.src_all = [torch.as_tensor(np.ascontiguousarray(s), **f64) for s in src]
        self.row_of_pt = torch.as_tensor(np.arange(self.n_points) - self.own_lo,
                                         dtype=torch.int32, device=dev)
        self.pt_idx = torch.arange(self.n_points, dtype=torch.int32, device=dev)
        self.c_rows = torch.as_tensor(self.c_idx - self.own_lo, dtype=torch.int32, device=dev)
        # per F-offset tables (contiguous [K] / [K, n_src])
        self.inv_dt_off, self.src_off, self.gidx_off = {}, [{}, {}], {}
        self.inv_dt_off_h = {}
        for j in range(1, self.m + 1):
            pts = self.c_idx - self.m + j
            pt = torch.as_tensor(pts, device=dev)
            self.inv_dt_off[j] = self.inv_dt_all[pt].contiguous()
            self.inv_dt_off_h[j] = np.ascontiguousarray(inv[pts])
            for sm in (0, 1):
                self.src_off[sm][j] = self.src_all[sm][pt].contiguous()
            self.gidx_off[j] = torch.as_tensor(pts - self.own_lo, dtype=torch.int32,
                                               device=dev)
        # sweep buffers
        self.start = torch.zeros(self.K, self.n, **f64)
        self.w = [torch.zeros(self.K, self.n, **f64), torch.zeros(self.K, self.n, **f64)]
        self.sumsq = torch.zeros(max(self.K, 1), **f64)
        self.loss = torch.zeros(max(self.K, 1), **f64)
        self.res = None


class MgritSolver:
    """Parallel-in-time solve of a GPU problem over a time hierarchy
    (reference mgrit.py:290-794)."""

    def __init__(self, problem, hierarchy, cycle=None, stopping=None, transport=None):
        t_setup = time.perf_counter()
        self.problem = problem
        self.hierarchy = hierarchy
        self.cycle = cycle if cycle is not None else CycleSpec()
        self.stopping = stopping if stopping is not None else StoppingCriterion()
        self.transport = transport if transport is not None else NullTransport()
        n_levels = hierarchy.n_levels
        if self.cycle.kind == "two-level" and n_levels > 2:
            n_levels = 2
        self.n_levels = n_levels
        self.assignment = assign_spatial_levels(self.cycle.spatial_strategy, n_levels,
                                                problem.spatial.n_grids)
        self.levels = [_Level(self, l, hierarchy[l], hierarchy.splittings[l],
                              self.assignment[l]) for l in range(n_levels)]
        dev = problem.device
        f64 = dict(dtype=torch.float64, device=dev)
        # fine-level transfer buffers (restriction targets on the next grid)
        for l in range(n_levels - 1):
            lvl, nxt = self.levels[l], self.levels[l + 1]
            lvl.res = torch.zeros(lvl.K, lvl.n, **f64)
            # restricted copies R(u_c), R(u_{c-1}) exist only across a change of
            # grid; on the same grid they are the C-store and the interval starts
            # themselves (17 GB less at config 4's level 0)
            if nxt.s != lvl.s:
                lvl.kept = torch.zeros(lvl.K, nxt.n, **f64)
                lvl.lkept = torch.zeros(lvl.K, nxt.n, **f64)
            else:
                lvl.kept = lvl.lkept = None
            lvl.cprop = torch.zeros(lvl.K, nxt.n, **f64)
            lvl.crhs = torch.zeros(lvl.K, nxt.n, **f64)
        # every distinct 1/dt of the levels on a grid, factored in one launch
        # per grid at setup (banded Cholesky) instead of at first use
        if hasattr(problem, "prefactor"):
            for s_lvl in sorted(set(self.assignment[:n_levels])):
                vals = [lv.inv_dt_all_h[1:] for lv in self.levels if lv.s == s_lvl]
                if vals:
                    problem.prefactor(s_lvl, np.unique(np.concatenate(vals)))
        self._plans = {}
        # CUDA-graph replay of the coarsest chain: problems opt in
        # (graph_safe: Phi launches with no host read); PINTGPU_GRAPHS=0 disables
        self._graphs = (bool(getattr(problem, "graph_safe", False))
                        and os.environ.get("PINTGPU_GRAPHS", "1") != "0")
        self._smooth = False
        self._probe_prop = None      # probe result reusable by the next level-0 FC sweep
        import inspect
        self._takes_host_dt = "inv_dt_host" in inspect.signature(problem.phi_batch).parameters
        # without the host copy of 1/dt Phi reads it back (a sync): not capturable
        self._graphs = self._graphs and self._takes_host_dt
        self.phi_columns = 0
        self.phi_calls = 0
        self.setup_seconds = time.perf_counter() - t_setup

    # --- storage accounting (reference mgrit.py:320-331) ---
    def storage_report(self):
        per = []
        for lvl in self.levels:
            c = lvl.K if not lvl.empty else len(lvl.decomp.c_points(self.transport.rank))
            if lvl.index > 0:
                c += 2 * lvl.n_owned
            per.append(c)
        est = storage_estimate(self.n_levels, self.hierarchy[0].n_steps,
                               self.hierarchy.factors[:self.n_levels - 1],
                               self.transport.size,
                               coarsest_factor=self.levels[-1].splitting.factor)
        return StorageReport(per_level=per, total=sum(per), estimate=est)

    # --- batched Phi wrappers ---
    def _phi_off(self, lvl, U, j, out, add_rhs=True):
        """Offset-j step of every owned interval: out = Phi(U) (+ rhs)."""
        use_g = add_rhs and lvl.use_rhs
        try:
            self.problem.phi_batch(lvl.s, U, lvl.inv_dt_off[j], lvl.src_off[self._smooth][j],
                                   out, g=lvl.rhs if use_g else None,
                                   g_idx=lvl.gidx_off[j] if use_g else None,
                                   **self._host_dt(lvl.inv_dt_off_h[j]))
        except NewtonConvergenceError as e:
            # t_next of the failing interval's step (problems.py:240-244)
            col = getattr(e, "column", -1)
            if 0 <= col < len(lvl.c_idx):
                e.at_time(lvl.t[lvl.c_idx[col] - lvl.m + j], lvl.s)
            raise
        self.phi_columns += U.shape[0]
        self.phi_calls += 1

    def _phi_pts(self, lvl, U, lo, hi, out, g=None, g_idx=None):
        """Consecutive points lo..hi-1 of lvl's grid, one column each."""
        try:
            self.problem.phi_batch(lvl.s, U, lvl.inv_dt_all[lo:hi],
                                   lvl.src_all[self._smooth][lo:hi], out, g=g, g_idx=g_idx,
                                   **self._host_dt(lvl.inv_dt_all_h[lo:hi]))
        except NewtonConvergenceError as e:
            col = getattr(e, "column", -1)
            if 0 <= col < hi - lo:
                e.at_time(lvl.t[lo + col], lvl.s)
            raise
        self.phi_columns += hi - lo
        self.phi_calls += 1

    def _host_dt(self, arr):
        """host copy of 1/dt for problems that accept it (skips a D2H read)"""
        return {"inv_dt_host": arr} if self._takes_host_dt else {}

    # --- communication (reference mgrit.py:339-357) ---
    def _exchange_left(self, lvl):
        """Send the last owned C-state (pre-sweep) right, receive the left
        boundary (mgrit.py:339-350).  The transfer is in flight until the
        returned boundary's ready(); _starts overlaps it with the
        copy of the interior interval starts, the only work of a sweep that
        does not depend on the boundary's batch."""
        d, r = lvl.decomp, self.transport.rank
        if lvl.empty:
            return None
        right, left = d.right_neighbor(r), d.left_neighbor(r)
        sends = [(right, lvl.c_store[-1])] if (right is not None and lvl.K) else []
        if left is None:
            return _Boundary(lvl.anchor, self.transport.exchange_async(sends, []))
        buf = torch.empty(lvl.n, dtype=torch.float64, device=self.problem.device)
        return _Boundary(buf, self.transport.exchange_async(sends, [(left, buf)]))

    def _starts(self, lvl, boundary):
        """Interval starts of a sweep: row 0 = the left boundary, row k = the
        pre-sweep C-value k - 1.  The interior rows are copied while the
        boundary exchange is still in flight."""
        if boundary is None:
            return lvl.start
        if lvl.K > 1:
            lvl.start[1:].copy_(lvl.c_store[:-1])
        buf = boundary.ready()
        if lvl.K:
            lvl.start[0].copy_(buf)
        return lvl.start

    def _walk(self, lvl, start):
        """F-walk of all owned intervals; returns the buffer with the last
        F-state of each interval (mgrit.py:368-376)."""
        cur = start
        for j in range(1, lvl.m):
            out = lvl.w[j & 1]
            self._phi_off(lvl, cur, j, out)
            cur = out
        return cur

    def _other(self, lvl, buf):
        return lvl.w[0] if buf is lvl.w[1] else lvl.w[1]

    # --- sweeps ---
    def _fc_sweep(self, lvl):
        """mgrit.py:378-393"""
        if lvl.index == 0 and self._probe_prop is not None:
            # The residual probe that precedes every cycle ran exactly this
            # F-walk and C-step from the same pre-sweep C-values (and sent the
            # same boundary): its propagated C-values are this sweep's result,
            # bit for bit, so the sweep is not recomputed.
            prop, self._probe_prop = self._probe_prop, None
            if prop is not False:
                lvl.c_store.copy_(prop)
            return
        self._probe_prop = None
        boundary = self._exchange_left(lvl)
        if lvl.empty or not lvl.K:
            _drain(boundary)
            return
        last_f = self._walk(lvl, self._starts(lvl, boundary))
        self._phi_off(lvl, last_f, lvl.m, lvl.c_store)

    def _plan(self, key, points, src, dst):
        if key not in self._plans:
            self._plans[key] = plan_moves(points, src, dst, self.transport.rank)
        return self._plans[key]

    def _restrict_plan(self, lvl, nxt):
        kf = lvl.splitting.n_intervals
        pts = np.arange(1, kf + 1)
        src = [lvl.decomp.unit_owner(j - 1) for j in pts]
        dst = [nxt.decomp.point_owner(j) for j in pts]
        return self._plan(("restrict", lvl.index), pts, src, dst)

    def _restrict_sweep(self, lvl, nxt):
        """mgrit.py:395-450"""
        self._probe_prop = None
        prob = self.problem
        coarsen = nxt.s != lvl.s
        boundary = self._exchange_left(lvl)
        if not lvl.empty and lvl.K:
            start = self._starts(lvl, boundary)
            last_f = self._walk(lvl, start)
            prop = self._other(lvl, last_f)
            self._phi_off(lvl, last_f, lvl.m, prop, add_rhs=False)
            use_g = lvl.use_rhs
            prob.c_residual(lvl.s, prop, lvl.c_store, lvl.sumsq,
                            g=lvl.rhs if use_g else None,
                            g_idx=lvl.gidx_off[lvl.m] if use_g else None, res=lvl.res)
            if coarsen:
                prob.restrict(lvl.s, lvl.c_store, lvl.kept)
                prob.restrict(lvl.s, start, lvl.lkept)
                kept, lkept = lvl.kept, lvl.lkept
            else:
                kept, lkept = lvl.c_store, start      # unchanged until the sweep ends
            j0 = lvl.first + 1
            self._phi_pts(nxt, lkept, j0, j0 + lvl.K, lvl.cprop)
            prob.fas_rhs(nxt.s, coarsen, kept, lvl.cprop, lvl.res, lvl.crhs)
        else:
            _drain(boundary)
        local, sends, recvs = self._restrict_plan(lvl, nxt)
        j0 = lvl.first + 1
        kept_rows = lvl.kept if coarsen else lvl.c_store
        for _, lo, hi in local:
            nxt.u_keep[lo - nxt.own_lo:hi - nxt.own_lo].copy_(kept_rows[lo - j0:hi - j0])
            nxt.rhs[lo - nxt.own_lo:hi - nxt.own_lo].copy_(lvl.crhs[lo - j0:hi - j0])
        if sends or recvs:
            s_ops, r_ops = [], []
            for peer, lo, hi in sends:
                s_ops += [(peer, kept_rows[lo - j0:hi - j0]), (peer, lvl.crhs[lo - j0:hi - j0])]
            tmp = []
            for peer, lo, hi in recvs:
                a = torch.empty(hi - lo, nxt.n, dtype=torch.float64, device=prob.device)
                b = torch.empty_like(a)
                r_ops += [(peer, a), (peer, b)]
                tmp.append((lo, hi, a, b))
            self.transport.exchange(s_ops, r_ops)
            for lo, hi, a, b in tmp:
                nxt.u_keep[lo - nxt.own_lo:hi - nxt.own_lo].copy_(a)
                nxt.rhs[lo - nxt.own_lo:hi - nxt.own_lo].copy_(b)
        nxt.use_rhs = True
        if nxt.K:
            prob.rows_axpby(nxt.K, nxt.c_store, nxt.u_keep, a_rows=nxt.c_rows)

    def _coarsest_solve(self, lvl, nested=False):
        """Gather, sequential on-device chain on rank 0, scatter
        (mgrit.py:452-495)."""
        prob, T = self.problem, self.transport
        dev = prob.device
        n_pts = lvl.n_points
        single = T.size == 1
        active = lvl.decomp.active_ranks()
        if single:
            g, g_idx = (lvl.rhs, lvl.row_of_pt) if lvl.use_rhs else (None, None)
        else:
            full = None
            if lvl.use_rhs:
                if T.rank == 0:
                    if lvl.full_rhs is None:
                        lvl.full_rhs = torch.zeros(n_pts, lvl.n, dtype=torch.float64, device=dev)
                    full = lvl.full_rhs
                    recvs = []
                    for w in active:
                        lo, hi = lvl.decomp.owned_range(w)
                        if w == 0:
                            full[lo:hi].copy_(lvl.rhs)
                        else:
                            recvs.append((w, full[lo:hi]))
                    T.exchange([], recvs)
                elif not lvl.empty:
                    T.exchange([(0, lvl.rhs)], [])
            g, g_idx = (full, lvl.pt_idx) if full is not None else (None, None)
        vals = None
        if T.rank == 0:
            vals = self._coarsest_chain(lvl, g, g_idx)
        # scatter
        if single:
            mine = vals[lvl.own_lo:lvl.own_hi]
        else:
            mine = None
            if T.rank == 0:
                sends = []
                for w in active:
                    lo, hi = lvl.decomp.owned_range(w)
                    if w == 0:
                        mine = vals[lo:hi]
                    else:
                        sends.append((w, vals[lo:hi]))
                T.exchange(sends, [])
            elif not lvl.empty:
                mine = torch.empty(lvl.n_owned, lvl.n, dtype=torch.float64, device=dev)
                T.exchange([], [(0, mine)])
        if lvl.empty:
            return
        if nested:
            lvl.u_keep.copy_(mine)
        else:
            prob.rows_axpby(lvl.n_owned, lvl.u_keep, mine, lvl.u_keep, sign=-1)   # v - kept
        if lvl.K:
            if nested:
                prob.rows_axpby(lvl.K, lvl.c_store, lvl.u_keep, a_rows=lvl.c_rows)
            else:
                prob.rows_axpby(lvl.K, lvl.c_store, lvl.c_store, lvl.u_keep, sign=1,
                                c_rows=lvl.c_rows)

    def _coarsest_chain(self, lvl, g, g_idx):
        """The serial chain v_i = Phi(v_{i-1}) (+ g_i) over the coarsest grid on
        rank 0 (mgrit.py:468-480): one single-column Phi per point, all on the
        device.  For problems whose Phi launches without host reads (linear,
        banded Cholesky) the chain of a level is captured into a CUDA graph the
        second time it runs -- same points, same factors, same buffers in every
        cycle -- and replayed afterwards, so later cycles pay one graph launch
        instead of ~10 kernel launches per point."""
        n_pts = lvl.n_points
        if lvl.chain_vals is None:
            lvl.chain_vals = torch.empty(n_pts, lvl.n, dtype=torch.float64,
                                         device=self.problem.device)
        vals = lvl.chain_vals
        vals[0].copy_(lvl.anchor)

        def run():
            for i in range(1, n_pts):
                self._phi_pts(lvl, vals[i - 1:i], i, i + 1, vals[i:i + 1],
                              g=g, g_idx=None if g is None else g_idx[i:i + 1])

        key = (self._smooth, None if g is None else g.data_ptr())
        entry = lvl.chain_graphs.get(key)
        if not self._graphs or n_pts < 3:
            run()
        elif entry is None:
            run()                                   # warms factors, spikes, groupings
            lvl.chain_graphs[key] = "warm"
        elif entry == "warm":
            graph = torch.cuda.CUDAGraph()
            calls, cols = self.phi_calls, self.phi_columns
            try:
                with torch.cuda.graph(graph, capture_error_mode="thread_local"):
                    run()
                lvl.chain_graphs[key] = (graph, self.phi_calls - calls,
                                         self.phi_columns - cols)
                graph.replay()
            except Exception:                       # not capturable here: stay eager
                self._graphs = False
                lvl.chain_graphs.clear()
                self.phi_calls, self.phi_columns = calls, cols
                torch.cuda.synchronize(self.problem.device)
                vals[0].copy_(lvl.anchor)
                run()
        else:
            graph, calls, cols = entry
            graph.replay()
            self.phi_calls += calls
            self.phi_columns += cols
        return vals

    def _ascend(self, coarse, fine, inject=False, solved=False):
        """mgrit.py:497-571: coarse walk (unless solved) turning u_keep into
        the payload v - kept (or v), then delivery to the fine C-store."""
        self._probe_prop = None
        prob = self.problem
        if not coarse.empty and not solved:
            boundary = self._exchange_left(coarse)
            m, K = coarse.m, coarse.K
            if not K:
                _drain(boundary)
            if K:
                cur = self._starts(coarse, boundary)
                for j in range(1, m + 1):
                    if j < m:
                        out = coarse.w[j & 1]
                        self._phi_off(coarse, cur, j, out)
                        cur = out
                    else:
                        cur = coarse.c_store
                    # rows j - 1, j - 1 + m, ... of u_keep: v (inject) or v - kept
                    if inject:
                        prob.rows_axpby(K, coarse.u_keep, cur, out_rows=(j - 1, m))
                    else:
                        prob.rows_axpby(K, coarse.u_keep, cur, coarse.u_keep, sign=-1,
                                        out_rows=(j - 1, m), c_rows=(j - 1, m))
            # F-tail after the last owned C-point (mgrit.py:529-532)
            last_c = int(coarse.c_idx[-1]) if K else coarse.left_index
            if coarse.own_hi - 1 > last_c:
                v = (coarse.c_store[-1] if K else boundary.ready()).reshape(1, -1).contiguous()
                for i in range(last_c + 1, coarse.own_hi):
                    out = torch.empty_like(v)
                    use_g = coarse.use_rhs
                    self._phi_pts(coarse, v, i, i + 1, out,
                                  g=coarse.rhs if use_g else None,
                                  g_idx=coarse.row_of_pt[i:i + 1] if use_g else None)
                    r = i - coarse.own_lo
                    if inject:
                        coarse.u_keep[r].copy_(out[0])
                    else:
                        prob.rows_axpby(1, coarse.u_keep, out, coarse.u_keep, sign=-1,
                                        out_rows=(r, 0), c_rows=(r, 0))
                    v = out
        self._deliver(coarse, fine, inject)

    def _deliver(self, coarse, fine, inject):
        prob = self.problem
        coarsen = coarse.s != fine.s
        key = ("ascend", coarse.index)
        if key not in self._plans:
            kf = fine.splitting.n_intervals
            pts = np.arange(1, min(coarse.n_points - 1, kf) + 1)
            src = [coarse.decomp.point_owner(i) for i in pts]
            dst = [fine.decomp.unit_owner(i - 1) for i in pts]
            self._plans[key] = plan_moves(pts, src, dst, self.transport.rank)
        local, sends, recvs = self._plans[key]

        def apply(lo, hi, payload):
            a, b = lo - 1 - fine.first, hi - 1 - fine.first
            dst = fine.c_store[a:b]
            if coarsen:
                prob.prolong_add(coarse.s, payload, dst, beta=0.0 if inject else 1.0)
            elif inject:
                dst.copy_(payload)
            else:
                prob.rows_axpby(b - a, dst, dst, payload, sign=1)

        for _, lo, hi in local:
            apply(lo, hi, coarse.u_keep[lo - coarse.own_lo:hi - coarse.own_lo])
        if sends or recvs:
            s_ops = [(peer, coarse.u_keep[lo - coarse.own_lo:hi - coarse.own_lo])
                     for peer, lo, hi in sends]
            tmp, r_ops = [], []
            for peer, lo, hi in recvs:
                a = torch.empty(hi - lo, coarse.n, dtype=torch.float64, device=prob.device)
                r_ops.append((peer, a))
                tmp.append((lo, hi, a))
            self.transport.exchange(s_ops, r_ops)
            for lo, hi, a in tmp:
                apply(lo, hi, a)

    def _probe(self, lvl):
        """mgrit.py:573-598: residual and per-C losses, state untouched."""
        prob = self.problem
        boundary = self._exchange_left(lvl)
        # idle ranks mark the reuse too, so every rank skips the same exchange
        self._probe_prop = (False if (lvl.index == 0 and not self._smooth and not lvl.use_rhs)
                            else None)
        if lvl.empty or not lvl.K:
            _drain(boundary)
            return 0.0, np.zeros(0)
        last_f = self._walk(lvl, self._starts(lvl, boundary))
        prop = self._other(lvl, last_f)
        self._phi_off(lvl, last_f, lvl.m, prop, add_rhs=False)
        if lvl.index == 0 and not lvl.use_rhs and not self._smooth:
            self._probe_prop = prop          # = the next cycle's first C-relaxation
        use_g = lvl.use_rhs
        prob.c_residual(lvl.s, prop, lvl.c_store, lvl.sumsq,
                        g=lvl.rhs if use_g else None,
                        g_idx=lvl.gidx_off[lvl.m] if use_g else None,
                        last_f=last_f, inv_dt=lvl.inv_dt_off[lvl.m], loss=lvl.loss)
        sq = lvl.sumsq[:lvl.K].cpu().numpy()
        total = 0.0
        for v in sq:                       # sequential, like mgrit.py:592
            total += float(v)
        return total, lvl.loss[:lvl.K].cpu().numpy().copy()

    # --- cycles (mgrit.py:602-635) ---
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
        self._ascend(self.levels[l + 1], self.levels[l], solved=(l + 1 == self.n_levels - 1))

    def _fcycle(self, l):
        if l == self.n_levels - 1:
            self._coarsest_solve(self.levels[l])
            return
        self._descend(l)
        self._fcycle(l + 1)
        self._ascend(self.levels[l + 1], self.levels[l], solved=(l + 1 == self.n_levels - 1))
        if l > 0:
            self._vcycle(l)

    def _iterate_once(self):
        if self.n_levels == 1:
            self._coarsest_solve_single()
        elif self.cycle.kind == "F":
            self._fcycle(0)
        else:
            self._vcycle(0)

    def _coarsest_solve_single(self):
        """mgrit.py:637-655: sequential walk depositing C-values."""
        self._probe_prop = None
        lvl = self.levels[0]
        if lvl.empty:
            return
        d, r = lvl.decomp, self.transport.rank
        left = d.left_neighbor(r)
        if left is None:
            v = lvl.anchor.reshape(1, -1).clone()
        else:
            v = torch.empty(1, lvl.n, dtype=torch.float64, device=self.problem.device)
            self.transport.exchange([], [(left, v[0])])
        c_set = {int(c): k for k, c in enumerate(lvl.c_idx)}
        for i in range(lvl.own_lo, lvl.own_hi):
            if lvl.K and i > int(lvl.c_idx[-1]):
                break
            out = torch.empty_like(v)
            self._phi_pts(lvl, v, i, i + 1, out)
            if i in c_set:
                lvl.c_store[c_set[i]].copy_(out[0])
            v = out
        right = d.right_neighbor(r)
        if right is not None and lvl.K:
            self.transport.exchange([(right, lvl.c_store[-1])], [])

    def _nested_iterations(self):
        """mgrit.py:659-675"""
        self._smooth = True
        try:
            bottom = self.levels[-1]
            if self.n_levels == 1:
                self._coarsest_solve_single()
                return
            bottom.use_rhs = False
            self._coarsest_solve(bottom, nested=True)
            for l in range(self.n_levels - 2, -1, -1):
                self._ascend(self.levels[l + 1], self.levels[l], inject=True,
                             solved=(l + 1 == self.n_levels - 1))
                if l > 0:
                    self.levels[l].use_rhs = False
                    self._vcycle(l)
        finally:
            self._smooth = False

    # --- driver (mgrit.py:679-761) ---
    def _initialize_guess(self):
        for lvl in self.levels:
            if lvl.K:
                self.problem.rows_axpby(lvl.K, lvl.c_store, lvl.anchor, a_rows=(0, 0))
            lvl.use_rhs = False

    def seed(self, trajectory):
        """Load the fine C-store from a full trajectory ([n_points, n] tensor
        or array, or a SpaceTimeVector)."""
        lvl = self.levels[0]
        if not lvl.K:
            return
        if hasattr(trajectory, "states"):
            rows = torch.stack([torch.cat([trajectory[int(c)].field.to(self.problem.device),
                                           torch.as_tensor(trajectory[int(c)].scalars,
                                                           device=self.problem.device)])
                                for c in lvl.c_idx])
        else:
            tr = torch.as_tensor(np.asarray(trajectory) if not torch.is_tensor(trajectory)
                                 else trajectory, device=self.problem.device)
            rows = tr[torch.as_tensor(lvl.c_idx, device=tr.device)]
        lvl.c_store.copy_(rows.to(self.problem.device, torch.float64))

    def _sync(self):
        if self.problem.device.type == "cuda":
            torch.cuda.synchronize(self.problem.device)

    def solve(self, gather_solution=True, initial_guess=None):
        T = self.transport
        run = SolverRun(n_workers=T.size)
        t_setup = time.perf_counter()
        self.phi_columns = 0          # per-solve counts (a solver object is reusable)
        self.phi_calls = 0
        self._initialize_guess()
        if initial_guess is not None:
            self.seed(initial_guess)
        elif self.cycle.nested_iterations and self.n_levels > 1:
            try:
                self._nested_iterations()
            except NewtonConvergenceError as e:
                if T.size > 1:
                    raise
                run.failure = str(e)
        self._sync()
        run.setup_seconds = self.setup_seconds + (time.perf_counter() - t_setup)
        t_solve = time.perf_counter()
        prev_losses = None
        if run.failure is None:
            try:
                run.initial_residual, prev_losses = self._measure()
            except NewtonConvergenceError as e:
                if T.size > 1:
                    raise
                run.failure = str(e)
        if run.failure is None:
            for it in range(1, self.cycle.max_iters + 1):
                try:
                    self._iterate_once()
                    norm, losses = self._measure()
                except NewtonConvergenceError as e:
                    if T.size > 1:
                        raise
                    run.failure = str(e)
                    break
                change = T.max(qoi_change(losses, prev_losses) if losses.size else 0.0)
                prev_losses = losses
                run.iterations = it
                run.residual_norms.append(norm)
                run.qoi_changes.append(change)
                run.iteration_seconds.append(time.perf_counter() - t_solve)
                if self.n_levels == 1:
                    run.converged = True
                    break
                value = norm if self.stopping.kind == "residual-norm" else change
                if value < self.stopping.tolerance:
                    run.converged = True
                    break
        self._sync()
        run.solve_seconds = time.perf_counter() - t_solve
        run.level_seconds = [lvl.seconds for lvl in self.levels]
        run.storage = self.storage_report()
        run.phi_columns = self.phi_columns
        run.phi_calls = self.phi_calls
        solution = None
        if gather_solution and run.failure is None:
            solution = self._materialize()
        return run, solution

    def _measure(self):
        sum_sq, losses = self._probe(self.levels[0])
        return self.transport.sum_ordered(sum_sq) ** 0.5, losses

    def _materialize(self):
        """Walk out the fine trajectory; rank 0 returns [n_points, n]
        (mgrit.py:763-794)."""
        lvl, T, dev = self.levels[0], self.transport, self.problem.device
        chunk = None
        if not lvl.empty:
            boundary = self._exchange_left(lvl)
            chunk = torch.empty(lvl.n_owned, lvl.n, dtype=torch.float64, device=dev)
            m, K = lvl.m, lvl.K
            if not K:
                _drain(boundary)
            if K:
                cur = self._starts(lvl, boundary)
                for j in range(1, m):
                    out = lvl.w[j & 1]
                    self._phi_off(lvl, cur, j, out)
                    chunk[j - 1::m][:K].copy_(out)
                    cur = out
                chunk[m - 1::m][:K].copy_(lvl.c_store)
            last_c = int(lvl.c_idx[-1]) if K else lvl.left_index
            v = (lvl.c_store[-1] if K else boundary.ready()).reshape(1, -1).contiguous()
            for i in range(last_c + 1, lvl.own_hi):
                out = torch.empty_like(v)
                self._phi_pts(lvl, v, i, i + 1, out)
                chunk[i - lvl.own_lo].copy_(out[0])
                v = out
        if T.size == 1:
            full = torch.empty(lvl.n_points, lvl.n, dtype=torch.float64, device=dev)
            full[0].copy_(lvl.anchor)
            full[lvl.own_lo:lvl.own_hi].copy_(chunk)
            return full
        if T.rank == 0:
            full = torch.empty(lvl.n_points, lvl.n, dtype=torch.float64, device=dev)
            full[0].copy_(lvl.anchor)
            recvs = []
            for w in lvl.decomp.active_ranks():
                lo, hi = lvl.decomp.owned_range(w)
                if w == 0:
                    full[lo:hi].copy_(chunk)
                else:
                    recvs.append((w, full[lo:hi]))
            T.exchange([], recvs)
            return full
        if chunk is not None:
            T.exchange([(0, chunk)], [])
        return None


def mgrit_solve(problem, hierarchy, cycle=None, stopping=None, transport=None,
                gather_solution=True, initial_guess=None):
    """reference mgrit.py:797-801"""
    solver = MgritSolver(problem, hierarchy, cycle, stopping, transport)
    return solver.solve(gather_solution=gather_solution, initial_guess=initial_guess)


def sequential_solve(problem, times, spatial_level=0, smooth=False):
    """GPU sequential time stepping (reference problems.py:319-339): the
    time-to-solution baseline.  Returns [n, size] device trajectory."""
    n = len(times)
    size = problem.state_size(spatial_level) if hasattr(problem, "state_size") \
        else problem.spatial.size(spatial_level)
    dev = problem.device
    out = torch.empty(n, size, dtype=torch.float64, device=dev)
    out[0].zero_()
    t = np.asarray(times, dtype=float)
    inv = torch.as_tensor(1.0 / (t[1:] - t[:-1]), dtype=torch.float64, device=dev)
    src = torch.as_tensor(np.ascontiguousarray(problem.source_values(t[1:], smooth)),
                          dtype=torch.float64, device=dev)
    for i in range(1, n):
        problem.phi_batch(spatial_level, out[i - 1:i], inv[i - 1:i], src[i - 1:i],
                          out[i:i + 1])
    return out
