"""The GPU problem object: the reference's Phi plug-in contract, batched.

Reference contract (problems.py:1-17, consumed by mgrit.py:361-366):

    step(u_prev, t_prev, t_next, spatial_level=0, guess=None, smooth=False)
        -> (BlockState, StepDiagnostics)
    initial_state(spatial_level), loss_weights(spatial_level), forcing(...),
    spatial (restrict_state / prolong_error), n_scalars

GpuFemProblem keeps that contract (step() is the B = 1 view) and adds the
batched entry points the B200 engine drives: phi_batch over [B][n] device
states, transfers, C-point residuals and the FAS right-hand side, all going
through libpintgpu's C ABI (include/pintgpu.h).  Construction fails when the
library or a CUDA device is missing -- there is no CPU path.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import NewtonConvergenceError, PintGpuError
from .excitation import Excitation
from .mesh import build_grids
from .spatial import SpatialHierarchy2D
from .state import BlockState


@dataclass(frozen=True)
class StepDiagnostics:
    """reference problems.py:33-36"""
    iterations: int
    converged: bool = True


def _np_ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


class GpuFemProblem:
    """2D P1 eddy-current problem (linear or Brauer-nonlinear) on one GPU."""

    n_scalars = 0

    def __init__(self, spec, device=None, rtol=None, max_iters=None,
                 check_every=16, inner=None):
        if spec.get("surrogate") and type(self) is GpuFemProblem:
            raise ValueError("spec carries a surrogate machine: use GpuSurrogateProblem "
                             "(or make_problem)")
        if not torch.cuda.is_available():
            raise PintGpuError("GpuFemProblem needs a CUDA device (no CPU fallback)")
        self.lib = _lib.load()
        self.spec = spec
        self.device = torch.device("cuda", torch.cuda.current_device()
                                   if device is None else device)
        self.spatial = SpatialHierarchy2D(spec["N"], spec.get("n_spatial_grids", 1),
                                          spec.get("restriction", "injection"),
                                          spec.get("prolongation", "bilinear"),
                                          ops=self)
        ex = spec.get("excitation")
        self.excitation = Excitation(**ex) if ex else None
        self.grids = build_grids(spec)
        self.phases = self.grids[0].phases
        self.n_src = len(self.phases)
        ctx = ctypes.c_void_p()
        rc = self.lib.pg_create(ctypes.byref(ctx), self.device.index)
        if rc != 0 or not ctx:
            raise PintGpuError(f"pg_create failed on device {self.device} (code {rc})")
        self.ctx = ctx
        self._keep = []
        for g in self.grids:
            self._add_level(g)
        inner_cfg = inner_spec = spec.get("inner", {})
        nl = spec.get("nonlinear") or {}
        nt = nl.get("newton", {})
        kind = inner if inner is not None else inner_cfg.get("kind", "pcg")
        if kind not in ("pcg", "cholesky"):
            raise ValueError(f"inner solver must be 'pcg' or 'cholesky', got {kind!r}")
        self.inner = kind
        self.opts = _lib.SolverOpts(
            inner=_lib.PG_INNER_CHOLESKY if kind == "cholesky" else _lib.PG_INNER_PCG,
            rtol=float(rtol if rtol is not None else inner_spec.get("rtol", 1e-13)),
            max_iters=int(max_iters if max_iters is not None
                          else inner_spec.get("max_iters", 20000)),
            check_every=int(check_every),
            newton_tol=float(nt.get("tol", 1e-11)),
            newton_max_iters=int(nt.get("max_iters", 25)),
            damping=float(nt.get("damping", 0.5)),
            max_halvings=int(nt.get("max_halvings", 8)),
            nu0=float(spec["nu0"]), k1=float(nl.get("k1", 0.0)),
            k2=float(nl.get("k2", 0.0)), k3=float(nl.get("k3", 1.0)),
            dt_merge_rtol=float(inner_spec.get("dt_merge_rtol", 0.0)),
            strips=int(bool(inner_spec.get("strips", True))))
        _lib.check(self.ctx, self.lib.pg_set_options(self.ctx, ctypes.byref(self.opts)),
                   "pg_set_options")
        self._weights = [torch.as_tensor(g.weights, device=self.device) for g in self.grids]
        self.nonlinear = bool(spec.get("nonlinear"))
        # Phi of a linear level with the banded factors launches kernels only
        # (no host read, no allocation once warm): safe to capture in a CUDA graph
        self.graph_safe = (not self.nonlinear and kind == "cholesky"
                           and type(self) is GpuFemProblem)

    def _add_level(self, g):
        arrays = dict(row_ptr=np.ascontiguousarray(g.row_ptr, np.int32),
                      col_idx=np.ascontiguousarray(g.col_idx, np.int32),
                      m_val=np.ascontiguousarray(g.m_val),
                      k_val=np.ascontiguousarray(g.k_val),
                      shapes=np.ascontiguousarray(g.shapes.reshape(-1)),
                      weights=np.ascontiguousarray(g.weights))
        d = _lib.LevelDesc()
        d.n, d.nnz, d.side = g.n, g.nnz, g.side
        d.row_ptr = _np_ptr(arrays["row_ptr"], ctypes.c_int32)
        d.col_idx = _np_ptr(arrays["col_idx"], ctypes.c_int32)
        d.m_val = _np_ptr(arrays["m_val"], ctypes.c_double)
        d.k_val = _np_ptr(arrays["k_val"], ctypes.c_double)
        d.n_src = len(g.phases)
        d.shapes = _np_ptr(arrays["shapes"], ctypes.c_double)
        d.weights = _np_ptr(arrays["weights"], ctypes.c_double)
        d.n_elem = g.n_elem
        if g.n_elem:
            for k in ("elem_dof", "elem_geo", "node_elem_ptr", "node_elem"):
                arrays[k] = np.ascontiguousarray(getattr(g, k))
            d.elem_dof = _np_ptr(arrays["elem_dof"], ctypes.c_int32)
            d.elem_geo = _np_ptr(arrays["elem_geo"], ctypes.c_double)
            d.node_elem_ptr = _np_ptr(arrays["node_elem_ptr"], ctypes.c_int32)
            d.node_elem = _np_ptr(arrays["node_elem"], ctypes.c_int32)
        if getattr(g, "k_pre", None) is not None:
            arrays["k_pre"] = np.ascontiguousarray(g.k_pre)
            d.k_pre_val = _np_ptr(arrays["k_pre"], ctypes.c_double)
        idx = self.lib.pg_add_level(self.ctx, ctypes.byref(d))
        if idx < 0:
            _lib.check(self.ctx, _lib.PG_EINVAL, "pg_add_level")

    def use_strips(self, on=True):
        """Switch the banded-Cholesky Phi of large grids between the strip
        solve (default) and the natural-order band solve (the reference's
        dpbtrs ordering); both are exact direct solves."""
        self.opts.strips = int(bool(on))
        _lib.check(self.ctx, self.lib.pg_set_options(self.ctx, ctypes.byref(self.opts)),
                   "pg_set_options")

    def close(self):
        if getattr(self, "ctx", None):
            torch.cuda.synchronize(self.device)
            self.lib.pg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- the reference contract ---------------------------------------------------
    def state_size(self, spatial_level=0):
        """Entries of one device state row ([field | scalars])."""
        return self.spatial.size(spatial_level) + self.n_scalars

    def initial_state(self, spatial_level=0):
        return BlockState.zeros(self.spatial.size(spatial_level), 0, spatial_level,
                                device=self.device)

    def loss_weights(self, spatial_level=0):
        return self._weights[spatial_level]

    def source_values(self, times, smooth=False):
        """[len(times), n_src] excitation values (host)."""
        times = np.atleast_1d(np.asarray(times, dtype=float))
        if self.excitation is None or not self.n_src:
            return np.zeros((len(times), self.n_src))
        return self.excitation.table(self.phases, times, smooth)

    def forcing(self, t, spatial_level=0, smooth=False):
        v = torch.as_tensor(self.source_values([t], smooth)[0], device=self.device)
        g = self.grids[spatial_level]
        return v @ torch.as_tensor(g.shapes, device=self.device)

    def step(self, u_prev, t_prev, t_next, spatial_level=0, guess=None, smooth=False):
        """One implicit-Euler step (reference problems.py:138-146)."""
        n = self.spatial.size(spatial_level)
        if u_prev.field.numel() != n:
            raise ValueError(f"state has {u_prev.field.numel()} entries, grid "
                             f"{spatial_level} has {n}")
        dt = float(t_next) - float(t_prev)
        inv_dt = torch.tensor([1.0 / dt], dtype=torch.float64, device=self.device)
        src = torch.as_tensor(self.source_values([t_next], smooth),
                              device=self.device).reshape(1, -1)
        u_in = u_prev.field.to(self.device).reshape(1, n).contiguous()
        gs = None
        if guess is not None and guess is not u_prev:
            gs = guess.field.to(self.device).reshape(1, n).contiguous()
        out = torch.empty(1, n, dtype=torch.float64, device=self.device)
        try:
            self.phi_batch(spatial_level, u_in, inv_dt, src, out, guess=gs)
        except NewtonConvergenceError as e:
            e.at_time(t_next, spatial_level)
            raise
        st = self.last_stats()
        if st["failed"]:
            raise PintGpuError(f"inner PCG did not converge at t={t_next:.6g} "
                               f"on grid {spatial_level}")
        its = st["newton_iters"] if self.nonlinear else st["batch_iters"]
        return (BlockState(out[0], spatial_level=spatial_level),
                StepDiagnostics(iterations=int(its)))

    # --- batched entry points -------------------------------------------------------
    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def phi_batch(self, level, u_prev, inv_dt, src, out, g=None, g_idx=None, guess=None,
                  inv_dt_host=None):
        """out[b] = Phi(u_prev[b]) (+ g[g_idx[b]]).  Device tensors: u_prev/out
        [B, n] fp64, inv_dt [B], src [B, n_src], g [*, n], g_idx [B] int32;
        inv_dt_host: optional contiguous fp64 numpy copy of inv_dt."""
        B = int(u_prev.shape[0])
        hp = None
        if inv_dt_host is not None:
            hp = inv_dt_host.ctypes.data_as(ctypes.c_void_p)
        def call():
            return self.lib.pg_phi_batch_h(self.ctx, int(level), B, _lib.ptr(u_prev),
                                           _lib.ptr(guess), _lib.ptr(inv_dt), hp,
                                           _lib.ptr(src) if self.n_src else None, _lib.ptr(out),
                                           _lib.ptr(g), _lib.ptr(g_idx), self._stream())
        rc = call()
        if rc == _lib.PG_ECUDA and b"out of memory" in (self.lib.pg_last_error(self.ctx) or b""):
            # the library allocates its workspaces with cudaMalloc: hand it the
            # blocks torch's caching allocator holds but does not use, once
            torch.cuda.synchronize(self.device)
            torch.cuda.empty_cache()
            rc = call()
        if rc == _lib.PG_ENEWTON:
            col, its = ctypes.c_int(), ctypes.c_int()
            self.lib.pg_newton_failure(self.ctx, ctypes.byref(col), ctypes.byref(its))
            msg = self.lib.pg_last_error(self.ctx).decode()
            # time = t_next of the failing column (reference problems.py:240-244):
            # the batch only knows its columns, so callers that know the
            # column's time (step(), the engine's sweeps) fill it in
            err = NewtonConvergenceError(msg, time=None, iterations=its.value)
            err.column = int(col.value)
            raise err
        _lib.check(self.ctx, rc, "pg_phi_batch")

    def prefactor(self, level, inv_dt_host):
        """Factor every distinct 1/dt of the list up front (banded Cholesky;
        one launch, one CTA per factor)."""
        arr = np.ascontiguousarray(np.asarray(inv_dt_host, dtype=np.float64))
        _lib.check(self.ctx, self.lib.pg_prefactor(
            self.ctx, int(level), int(arr.size), arr.ctypes.data_as(ctypes.c_void_p),
            self._stream()), "pg_prefactor")

    def last_stats(self):
        s = _lib.PhiStats()
        _lib.check(self.ctx, self.lib.pg_last_stats(self.ctx, ctypes.byref(s)), "pg_last_stats")
        return {k: int(getattr(s, k)) for k, _ in s._fields_}

    def total_stats(self, reset=False):
        s = _lib.PhiStats()
        _lib.check(self.ctx, self.lib.pg_total_stats(self.ctx, ctypes.byref(s), int(reset)),
                   "pg_total_stats")
        return {k: int(getattr(s, k)) for k, _ in s._fields_}

    def profile(self, on=True):
        _lib.check(self.ctx, self.lib.pg_profile(self.ctx, int(bool(on))), "pg_profile")

    def profile_read(self, reset=False):
        arr = (_lib.KernelProfile * _lib.PG_PROFILE_KINDS)()
        _lib.check(self.ctx, self.lib.pg_profile_read(self.ctx, arr, _lib.PG_PROFILE_KINDS,
                                                      int(reset)),
                   "pg_profile_read")
        return [dict(name=a.name.decode(), total_ms=a.total_ms, launches=int(a.launches),
                     alg_bytes=a.alg_bytes, alg_flops=a.alg_flops,
                     column_iters=int(a.column_iters)) for a in arr]

    def launch_count(self):
        return int(self.lib.pg_launch_count(self.ctx))

    def restrict(self, fine_level, x, out):
        _lib.check(self.ctx, self.lib.pg_restrict(
            self.ctx, int(fine_level), int(x.shape[0]), _lib.ptr(x), _lib.ptr(out),
            self.spatial.r_mode, self._stream()), "pg_restrict")

    def prolong_add(self, coarse_level, x, out, out_idx=None, beta=1.0):
        _lib.check(self.ctx, self.lib.pg_prolong_add(
            self.ctx, int(coarse_level), int(x.shape[0]), _lib.ptr(x), _lib.ptr(out),
            _lib.ptr(out_idx), float(beta), self.spatial.p_mode, self._stream()),
            "pg_prolong_add")

    def c_residual(self, level, prop, c, sumsq, c_idx=None, g=None, g_idx=None,
                   res=None, last_f=None, inv_dt=None, loss=None):
        _lib.check(self.ctx, self.lib.pg_c_residual(
            self.ctx, int(level), int(prop.shape[0]), _lib.ptr(prop), _lib.ptr(c),
            _lib.ptr(c_idx), _lib.ptr(g), _lib.ptr(g_idx), _lib.ptr(res), _lib.ptr(sumsq),
            _lib.ptr(last_f), _lib.ptr(inv_dt), _lib.ptr(loss), self._stream()),
            "pg_c_residual")

    def rows_axpby(self, B, out, a, c=None, sign=1, out_rows=None, a_rows=None, c_rows=None):
        """out[ro(b)] = a[ra(b)] (+ sign * c[rc(b)]) for b < B over rows of
        equal length (2-D row-contiguous tensors, or one row).  A row selector
        is None (row b), an int32 device index tensor, or a (start, step) pair."""
        def sel(r):
            if r is None:
                return None, 0, 1
            if isinstance(r, tuple):
                return None, int(r[0]), int(r[1])
            return r, 0, 0
        ai, a0, a1 = sel(a_rows)
        ci, c0, c1 = sel(c_rows)
        oi, o0, o1 = sel(out_rows)
        _lib.check(self.ctx, self.lib.pg_rows_axpby(
            self.ctx, int(out.shape[-1]), int(B), _lib.ptr(a), _lib.ptr(ai), a0, a1,
            _lib.ptr(c), _lib.ptr(ci), c0, c1, int(sign), _lib.ptr(out), _lib.ptr(oi), o0, o1,
            self._stream()), "pg_rows_axpby")

    def fas_rhs(self, coarse_level, coarsen, kept, cprop, res, out):
        _lib.check(self.ctx, self.lib.pg_fas_rhs(
            self.ctx, int(coarse_level), int(bool(coarsen)), int(kept.shape[0]),
            _lib.ptr(kept), _lib.ptr(cprop), _lib.ptr(res), _lib.ptr(out),
            self.spatial.r_mode, self._stream()), "pg_fas_rhs")


class GpuSurrogateProblem(GpuFemProblem):
    """Rotor angle / speed one-way coupled to the field: reference
    problems.py:247-287 (SurrogateMachineProblem) on the 2D model.  The field
    takes the base problem's step (linear or Brauer-Newton, same kernels),
    then per column

        T = c . u_new,  omega' = (omega + dt T / I) / (1 + dt friction / I),
        theta' = theta + dt omega',

    with c = sin(2 pi x) h^2 (configs.with_surrogate).  Device states are
    augmented rows [field | theta, omega] (state_size = n + 2): norms include
    the scalars, transfers pass them through bitwise (spatial.py:64-84); the
    field part runs through the C ABI on packed copies, the scalars are
    column-wise torch ops."""

    n_scalars = 2

    def __init__(self, spec, **kw):
        sg = spec.get("surrogate") or {}
        self.inertia = float(sg.get("inertia", 1.0))
        self.friction = float(sg.get("friction", 0.1))
        if self.inertia <= 0.0 or self.friction < 0.0:
            raise ValueError("need inertia > 0 and friction >= 0")
        super().__init__(spec, **kw)
        self._coupling = [torch.as_tensor(g.coupling, device=self.device) for g in self.grids]

    def initial_state(self, spatial_level=0):
        return BlockState.zeros(self.spatial.size(spatial_level), 2, spatial_level,
                                device=self.device)

    def torque(self, field, spatial_level=0):
        return float(self._coupling[spatial_level] @ field.to(self.device))

    def step(self, u_prev, t_prev, t_next, spatial_level=0, guess=None, smooth=False):
        n = self.spatial.size(spatial_level)
        if u_prev.field.numel() != n or len(u_prev.scalars) != 2:
            raise ValueError(f"state needs {n} field entries and 2 scalars")
        dt = float(t_next) - float(t_prev)
        inv_dt = torch.tensor([1.0 / dt], dtype=torch.float64, device=self.device)
        src = torch.as_tensor(self.source_values([t_next], smooth),
                              device=self.device).reshape(1, -1)
        row = torch.empty(1, n + 2, dtype=torch.float64, device=self.device)
        row[0, :n] = u_prev.field.to(self.device)
        row[0, n:] = torch.as_tensor(u_prev.scalars, device=self.device)
        gs = None
        if guess is not None and guess is not u_prev:
            gs = torch.zeros_like(row)
            gs[0, :n] = guess.field.to(self.device)
        out = torch.empty_like(row)
        self.phi_batch(spatial_level, row, inv_dt, src, out, guess=gs, dt_host=[dt])
        st = self.last_stats()
        its = st["newton_iters"] if self.nonlinear else st["batch_iters"]
        return (BlockState(out[0, :n].clone(), out[0, n:].cpu().numpy(), spatial_level),
                StepDiagnostics(iterations=int(its)))

    def phi_batch(self, level, u_prev, inv_dt, src, out, g=None, g_idx=None, guess=None,
                  inv_dt_host=None, dt_host=None):
        n = self.spatial.size(level)
        B = int(u_prev.shape[0])
        uf = u_prev[:, :n].contiguous()
        sc = u_prev[:, n:].clone()                     # out may alias u_prev
        gf = guess[:, :n].contiguous() if guess is not None else None
        of = torch.empty(B, n, dtype=torch.float64, device=self.device)
        super().phi_batch(level, uf, inv_dt, src, of, guess=gf, inv_dt_host=inv_dt_host)
        if dt_host is not None:
            dt = torch.as_tensor(np.asarray(dt_host, dtype=float), device=self.device)
        elif inv_dt_host is not None:
            dt = torch.as_tensor(1.0 / np.asarray(inv_dt_host, dtype=float), device=self.device)
        else:
            dt = 1.0 / inv_dt
        T = of @ self._coupling[level]
        omega = (sc[:, 1] + dt * T / self.inertia) / (1.0 + dt * self.friction / self.inertia)
        theta = sc[:, 0] + dt * omega
        out[:, :n] = of
        out[:, n] = theta
        out[:, n + 1] = omega
        if g is not None:                              # u.add_scaled(g_i), mgrit.py:372-375
            if g_idx is None:
                out += g[:B]
            else:
                sel = g_idx.long()
                rows = (sel >= 0).nonzero().flatten()
                if rows.numel():
                    out[rows] += g[sel[rows]]

    def restrict(self, fine_level, x, out):
        nf, nc = self.spatial.size(fine_level), self.spatial.size(fine_level + 1)
        of = torch.empty(x.shape[0], nc, dtype=torch.float64, device=self.device)
        super().restrict(fine_level, x[:, :nf].contiguous(), of)
        out[:, :nc] = of
        out[:, nc:] = x[:, nf:]

    def prolong_add(self, coarse_level, x, out, out_idx=None, beta=1.0):
        nc, nf = self.spatial.size(coarse_level), self.spatial.size(coarse_level - 1)
        B = int(x.shape[0])
        tmp = torch.empty(B, nf, dtype=torch.float64, device=self.device)
        super().prolong_add(coarse_level, x[:, :nc].contiguous(), tmp, None, 0.0)
        rows = out_idx.long() if out_idx is not None else torch.arange(B, device=self.device)
        if beta == 0.0:
            out[rows, :nf] = tmp
            out[rows, nf:] = x[:, nc:]
        else:
            out[rows, :nf] += tmp
            out[rows, nf:] += x[:, nc:]

    def c_residual(self, level, prop, c, sumsq, c_idx=None, g=None, g_idx=None,
                   res=None, last_f=None, inv_dt=None, loss=None):
        n = self.spatial.size(level)
        B = int(prop.shape[0])
        cs = c[c_idx.long()] if c_idx is not None else c[:B]
        rf = torch.empty(B, n, dtype=torch.float64, device=self.device) if res is not None else None
        super().c_residual(level, prop[:, :n].contiguous(), cs[:, :n].contiguous(), sumsq,
                           None, g[:, :n].contiguous() if g is not None else None, g_idx,
                           rf, last_f[:, :n].contiguous() if last_f is not None else None,
                           inv_dt, loss)
        rs = prop[:, n:] - cs[:, n:]
        if g is not None:
            if g_idx is None:
                rs = rs + g[:B, n:]
            else:
                sel = g_idx.long()
                ok = sel >= 0
                gs = torch.zeros_like(rs)
                gs[ok] = g[sel[ok], n:]
                rs = torch.where(ok[:, None], rs + gs, rs)
        sumsq[:B] += rs[:, 0] * rs[:, 0] + rs[:, 1] * rs[:, 1]   # norm_sq, state.py:74-75
        if res is not None:
            res[:, :n] = rf
            res[:, n:] = rs

    def fas_rhs(self, coarse_level, coarsen, kept, cprop, res, out):
        nc = self.spatial.size(coarse_level)
        nf = self.spatial.size(coarse_level - 1) if coarsen else nc
        B = int(kept.shape[0])
        of = torch.empty(B, nc, dtype=torch.float64, device=self.device)
        super().fas_rhs(coarse_level, coarsen, kept[:, :nc].contiguous(),
                        cprop[:, :nc].contiguous(), res[:, :nf].contiguous(), of)
        out[:, :nc] = of
        out[:, nc:] = (kept[:, nc:] - cprop[:, nc:]) + res[:, nf:]


def make_problem(spec, **kw):
    """GpuSurrogateProblem for specs with a surrogate machine, else GpuFemProblem."""
    cls = GpuSurrogateProblem if spec.get("surrogate") else GpuFemProblem
    return cls(spec, **kw)
