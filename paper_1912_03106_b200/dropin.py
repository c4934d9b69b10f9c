"""Drop-in pieces for a reference-side caller (route A).

Two things a `pintmg` maintainer needs to put the B200 Phi behind the
reference's own engine:

* `OperatorLevel` / `GpuOperatorProblem` -- a GPU problem built from explicit
  operators (CSR of M_sigma and K_nu, load vectors) instead of a 2D model
  spec.  This is how the reference's own 1D `LinearDiffusionProblem`
  (problems.py:111-146: sigma/dt I + nu/dx^2 tridiag(-1, 2, -1)) runs through
  `pg_phi_batch`; `reference_1d_levels` builds exactly that operator.
* `ReferenceProblemAdapter` -- wraps any GPU problem so that an engine written
  against the reference contract (problems.py:1-17: numpy BlockState in,
  fresh numpy BlockState out, StepDiagnostics) can call it one interval at a
  time, as `MgritSolver._step` does (mgrit.py:361-366).

Neither has a CPU path: construction needs the CUDA library and a device.
"""

import ctypes
from types import SimpleNamespace

import numpy as np
import torch

from . import _lib
from .errors import PintGpuError
from .problem import GpuFemProblem, StepDiagnostics


def OperatorLevel(row_ptr, col_idx, m_val, k_val, shapes=None, weights=None, side=0):
    """One spatial grid given by its operators (host numpy arrays): CSR of the
    union pattern of M and K (columns sorted per row, diagonal present),
    load vectors shapes[n_src][n], Joule-loss weights[n]."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    n = int(row_ptr.size - 1)
    shapes = np.zeros((0, n)) if shapes is None else np.atleast_2d(np.asarray(shapes, float))
    if shapes.shape[1] != n:
        raise ValueError(f"shapes must be [n_src][{n}], got {shapes.shape}")
    return SimpleNamespace(
        n=n, nnz=int(col_idx.size), side=int(side), row_ptr=row_ptr, col_idx=col_idx,
        m_val=np.ascontiguousarray(m_val, dtype=np.float64),
        k_val=np.ascontiguousarray(k_val, dtype=np.float64),
        shapes=np.ascontiguousarray(shapes), phases=list(range(shapes.shape[0])),
        weights=np.ascontiguousarray(np.ones(n) if weights is None else weights, np.float64),
        n_elem=0, k_pre=None)


def reference_1d_levels(nx, n_grids=1, diffusivity=1.0, mass_coeff=1.0, shape=None):
    """The reference's 1D finite-difference operator on every grid of its
    nested hierarchy (spatial.py:20-39: n_coarse = (n_fine - 1) / 2, spacing
    1 / (n + 1)): M = mass_coeff I and K = diffusivity / dx^2 tridiag(-1, 2, -1)
    on the tridiagonal pattern; one load vector per grid, `shape(x)` sampled at
    the interior points (default sin(pi x), the reference's "sine" profile);
    loss weights mass_coeff dx (problems.py:99-101)."""
    levels = []
    n = int(nx)
    for g in range(n_grids):
        if g:
            if n % 2 == 0 or n < 3:
                raise ValueError(f"a {n}-point grid has no nested coarse grid")
            n = (n - 1) // 2
        dx = 1.0 / (n + 1)
        rows, cols, mv, kv = [0], [], [], []
        off, dia = -diffusivity / dx ** 2, 2.0 * diffusivity / dx ** 2
        for i in range(n):
            for j in (i - 1, i, i + 1):
                if 0 <= j < n:
                    cols.append(j)
                    mv.append(mass_coeff if j == i else 0.0)
                    kv.append(dia if j == i else off)
            rows.append(len(cols))
        x = np.arange(1, n + 1) * dx
        s = np.sin(np.pi * x) if shape is None else np.asarray(shape(x), float)
        levels.append(OperatorLevel(rows, cols, mv, kv, shapes=s[None, :],
                                    weights=np.full(n, mass_coeff * dx)))
    return levels


class _Grids1D:
    """Sizes of an operator hierarchy (the part of reference
    SpatialHierarchy the engine reads); the device transfer kernels are 2D
    tensor-product stencils, so operator problems run without spatial
    coarsening (spatial_strategy "none")."""

    restriction, prolongation, r_mode, p_mode = "injection", "bilinear", 0, 0

    def __init__(self, sizes):
        self.sizes = tuple(int(s) for s in sizes)

    @property
    def n_grids(self):
        return len(self.sizes)

    def size(self, grid):
        return self.sizes[grid]

    def spacing(self, grid):
        return 1.0 / (self.sizes[grid] + 1)

    def restrict_state(self, state):
        raise PintGpuError("operator problems have no device transfers (use "
                           "spatial_strategy='none')")

    prolong_error = restrict_state


class GpuOperatorProblem(GpuFemProblem):
    """Linear Phi for operators handed over as CSR: column b solves
    (inv_dt_b M + K) u = inv_dt_b M u_prev + sum_s v_s(t_b) shape_s through the
    same C ABI and kernels as the 2D model (banded Cholesky when
    inner="cholesky", Jacobi-PCG when "pcg").

    levels:  list of OperatorLevel
    source:  callable(times[k], smooth) -> [k][n_src] source values (None = 0)
    """

    def __init__(self, levels, source=None, device=None, inner="cholesky", rtol=1e-13,
                 max_iters=20000, check_every=16):
        if not torch.cuda.is_available():
            raise PintGpuError("GpuOperatorProblem needs a CUDA device (no CPU fallback)")
        if inner not in ("pcg", "cholesky"):
            raise ValueError(f"inner solver must be 'pcg' or 'cholesky', got {inner!r}")
        self.lib = _lib.load()
        self.spec = {"name": "operators"}
        self.device = torch.device("cuda", torch.cuda.current_device()
                                   if device is None else device)
        self.grids = list(levels)
        self.spatial = _Grids1D([g.n for g in self.grids])
        self.excitation = None
        self._source = source
        self.phases = self.grids[0].phases
        self.n_src = len(self.phases)
        ctx = ctypes.c_void_p()
        rc = self.lib.pg_create(ctypes.byref(ctx), self.device.index)
        if rc != 0 or not ctx:
            raise PintGpuError(f"pg_create failed on device {self.device} (code {rc})")
        self.ctx = ctx
        for g in self.grids:
            self._add_level(g)
        self.inner = inner
        self.opts = _lib.SolverOpts(
            inner=_lib.PG_INNER_CHOLESKY if inner == "cholesky" else _lib.PG_INNER_PCG,
            rtol=float(rtol), max_iters=int(max_iters), check_every=int(check_every),
            newton_tol=1e-11, newton_max_iters=25, damping=0.5, max_halvings=8,
            nu0=1.0, k1=0.0, k2=0.0, k3=1.0, dt_merge_rtol=0.0, strips=1)
        _lib.check(self.ctx, self.lib.pg_set_options(self.ctx, ctypes.byref(self.opts)),
                   "pg_set_options")
        self._weights = [torch.as_tensor(g.weights, device=self.device) for g in self.grids]
        self.nonlinear = False

    def source_values(self, times, smooth=False):
        times = np.atleast_1d(np.asarray(times, dtype=float))
        if self._source is None or not self.n_src:
            return np.zeros((len(times), self.n_src))
        v = np.asarray(self._source(times, smooth), dtype=float)
        return np.ascontiguousarray(v.reshape(len(times), self.n_src))


class ReferenceProblemAdapter:
    """A GPU problem behind the reference's problem contract (problems.py:1-17)
    for engines that hold host numpy states: `step` takes and returns the
    caller's own BlockState class (any class constructed as
    state_cls(field, scalars=None, spatial_level=0) with .field / .scalars /
    .spatial_level), one pg_phi_batch call with B = 1 per step -- the loop
    MgritSolver._step runs (mgrit.py:361-366).  Inputs are never mutated or
    aliased; Newton failures surface as the GPU problem's
    NewtonConvergenceError(message, time, iterations) (errors.py:4-10)."""

    def __init__(self, gpu_problem, state_cls, diag_cls=StepDiagnostics):
        self.gpu = gpu_problem
        self.state_cls = state_cls
        self.diag_cls = diag_cls
        self.n_scalars = int(getattr(gpu_problem, "n_scalars", 0))
        self.spatial = gpu_problem.spatial
        self.calls = 0

    def initial_state(self, spatial_level=0):
        n = self.gpu.spatial.size(spatial_level)
        return self.state_cls(np.zeros(n), np.zeros(self.n_scalars), spatial_level)

    def loss_weights(self, spatial_level=0):
        return self.gpu.loss_weights(spatial_level).cpu().numpy()

    def forcing(self, t, spatial_level=0, smooth=False):
        return self.gpu.forcing(t, spatial_level, smooth).cpu().numpy()

    def step(self, u_prev, t_prev, t_next, spatial_level=0, guess=None, smooth=False):
        p = self.gpu
        n = p.spatial.size(spatial_level)
        field = np.asarray(u_prev.field, dtype=np.float64)
        if field.size != n:
            raise ValueError(f"state has {field.size} entries, grid {spatial_level} has {n}")
        dev = p.device
        u = torch.as_tensor(field, device=dev).reshape(1, n).contiguous()
        gs = None
        if guess is not None and guess is not u_prev:
            gs = torch.as_tensor(np.asarray(guess.field, np.float64),
                                 device=dev).reshape(1, n).contiguous()
        inv = np.array([1.0 / (float(t_next) - float(t_prev))])
        inv_dt = torch.as_tensor(inv, device=dev)
        src = torch.as_tensor(p.source_values([t_next], smooth), device=dev).reshape(1, -1)
        out = torch.empty_like(u)
        try:
            p.phi_batch(spatial_level, u, inv_dt, src, out, guess=gs, inv_dt_host=inv)
        except Exception as e:                      # NewtonConvergenceError: fill in the time
            if hasattr(e, "at_time"):
                e.at_time(t_next, spatial_level)
            raise
        self.calls += 1
        its = 1
        if getattr(p, "nonlinear", False):
            its = int(p.last_stats()["newton_iters"])
        return (self.state_cls(out[0].cpu().numpy(), np.zeros(self.n_scalars), spatial_level),
                self.diag_cls(iterations=its))
