"""2D P1 magnetoquasistatic Phi on the unit square (oracle).

Model (BASELINE.json configs; decisions G1-G10 of SURVEY.md 8.0, written
down in DESIGN.md 2):

    sigma dA/dt - div(nu grad A) = J(t),  A = 0 on the boundary,

P1 triangles on an N x N cell grid, every cell cut along its '/' diagonal,
(N-1)^2 interior unknowns.  Per element (centroid rule): sigma = sigma_disc
inside the centred disc, 0 outside, plus sigma_reg everywhere; nu = nu0, or
in the nonlinear model nu0 (k1 exp(k2 |B|^2) + k3) in the iron annulus
(excluding source boxes), |B| = |grad A|.  J(t) = sum_phase v_phase(t) *
shape_phase with shape_phase the consistent load vector of the phase's
source boxes (amplitude and sign folded in) -- the 2D form of the
reference's `forcing = v(t) * shape` (problems.py:103-108).

Implicit Euler step (problems.py:8, :138-146):
    (M_sigma / dt + K) u = f(t_next) + M_sigma / dt u_prev,
solved by banded Cholesky (scipy cholesky_banded / cho_solve_banded, the
reference's own LAPACK path, problems.py:25, :130-146), factors cached per
(spatial_level, float(dt)).  Nonlinear: damped Newton restating
problems.py:201-244 with a banded Jacobian factorised per Newton iteration.

This assembly is an element loop written from the textbook P1 formulas; the
product assembles the same matrices independently (stencil form).
"""

import math

import numpy as np
import scipy.sparse as sp
from scipy.linalg import cho_solve_banded, cholesky_banded

from .excitation import Excitation
from .spatial2d import SpatialHierarchy2D
from .state import BlockState, SpaceTimeVector

MU0 = 4e-7 * math.pi


class NewtonConvergenceError(RuntimeError):
    """reference errors.py:4-10"""

    def __init__(self, message, time=None, iterations=None):
        super().__init__(message)
        self.time = time
        self.iterations = iterations


class StepDiagnostics:
    __slots__ = ("iterations", "converged")

    def __init__(self, iterations, converged=True):
        self.iterations = iterations
        self.converged = converged


# --- mesh and element data ---------------------------------------------------

class Mesh:
    """Structured '/'-diagonal P1 triangulation, interior-node numbering."""

    def __init__(self, n_cells):
        N = int(n_cells)
        self.N = N
        self.side = N - 1
        self.n = (N - 1) ** 2
        h = 1.0 / N
        tris = []
        for j in range(N):
            for i in range(N):
                a, b = (i, j), (i + 1, j)
                c, d = (i + 1, j + 1), (i, j + 1)
                tris.append((a, b, c))   # lower triangle
                tris.append((a, c, d))   # upper triangle
        self.tri_ij = np.array(tris, dtype=np.int64)          # (ne, 3, 2)
        xy = self.tri_ij * h
        self.xy = xy
        self.centroid = xy.mean(axis=1)
        x1, y1 = xy[:, 0, 0], xy[:, 0, 1]
        x2, y2 = xy[:, 1, 0], xy[:, 1, 1]
        x3, y3 = xy[:, 2, 0], xy[:, 2, 1]
        det = (x2 - x1) * (y3 - y1) - (x3 - x1) * (y2 - y1)
        self.area = 0.5 * np.abs(det)
        # gradients of the barycentric functions: b_i = (y_j - y_k) / det
        self.gb = np.stack([(y2 - y3), (y3 - y1), (y1 - y2)], axis=1) / det[:, None]
        self.gc = np.stack([(x3 - x2), (x1 - x3), (x2 - x1)], axis=1) / det[:, None]
        ii, jj = self.tri_ij[..., 0], self.tri_ij[..., 1]
        interior = (ii > 0) & (ii < N) & (jj > 0) & (jj < N)
        self.dof = np.where(interior, (jj - 1) * (N - 1) + (ii - 1), -1)

    def assemble(self, elem_mats):
        """Sum (ne, 3, 3) element matrices into an interior CSR matrix."""
        rows, cols, vals = [], [], []
        for a in range(3):
            for b in range(3):
                ok = (self.dof[:, a] >= 0) & (self.dof[:, b] >= 0)
                rows.append(self.dof[ok, a])
                cols.append(self.dof[ok, b])
                vals.append(elem_mats[ok, a, b])
        A = sp.coo_matrix((np.concatenate(vals),
                           (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.n, self.n)).tocsr()
        A.sum_duplicates()
        return A

    def assemble_vec(self, elem_vecs):
        out = np.zeros(self.n)
        for a in range(3):
            ok = self.dof[:, a] >= 0
            np.add.at(out, self.dof[ok, a], elem_vecs[ok, a])
        return out

    def stiffness_elem(self, nu):
        G = (self.gb[:, :, None] * self.gb[:, None, :]
             + self.gc[:, :, None] * self.gc[:, None, :])
        return (nu * self.area)[:, None, None] * G

    def mass_elem(self, sigma):
        base = np.full((3, 3), 1.0) + np.eye(3)
        return (sigma * self.area / 12.0)[:, None, None] * base[None]


def in_box(xy, box):
    x0, y0, x1, y1 = box
    return (xy[:, 0] >= x0) & (xy[:, 0] < x1) & (xy[:, 1] >= y0) & (xy[:, 1] < y1)


class LevelModel:
    """Matrices, source shapes and material maps of one spatial grid."""

    def __init__(self, spec, n_cells):
        self.mesh = mesh = Mesh(n_cells)
        c = mesh.centroid
        cx, cy = spec.get("disc_center", (0.5, 0.5))
        r2 = (c[:, 0] - cx) ** 2 + (c[:, 1] - cy) ** 2
        sigma = np.where(r2 < spec["disc_radius"] ** 2, spec["sigma_disc"], 0.0)
        sigma = sigma + spec["sigma_reg"]
        self.sigma = sigma
        self.nu0 = spec["nu0"]
        self.M = mesh.assemble(mesh.mass_elem(sigma))
        in_src = np.zeros(len(c), dtype=bool)
        phases = sorted({s["phase"] for s in spec["sources"]})
        self.phases = phases
        shapes = []
        for ph in phases:
            load = np.zeros(len(c))
            for s in spec["sources"]:
                if s["phase"] != ph:
                    continue
                inside = in_box(c, s["box"])
                in_src |= inside
                load += np.where(inside, s["sign"] * spec["amplitude"], 0.0)
            shapes.append(mesh.assemble_vec(
                (load * mesh.area / 3.0)[:, None] * np.ones((1, 3))))
        self.shapes = np.array(shapes)
        nl = spec.get("nonlinear")
        if nl:
            r = np.sqrt(r2)
            self.iron = (r >= nl["r_in"]) & (r <= nl["r_out"]) & ~in_src
            self.k1, self.k2, self.k3 = nl["k1"], nl["k2"], nl["k3"]
        else:
            self.iron = np.zeros(len(c), dtype=bool)
        self.K = mesh.assemble(mesh.stiffness_elem(np.full(len(c), self.nu0)))
        self.lumped = np.asarray(self.M.sum(axis=1)).ravel()
        self.bw = mesh.side + 1   # '/' diagonal neighbour is +(N-1)+1

    # nonlinear pieces (2D form of problems.py:149-199)
    def gradients(self, u):
        ue = np.where(self.mesh.dof >= 0, u[np.maximum(self.mesh.dof, 0)], 0.0)
        gx = np.sum(self.mesh.gb * ue, axis=1)
        gy = np.sum(self.mesh.gc * ue, axis=1)
        return gx, gy

    def nu(self, s2):
        e = np.exp(self.k2 * s2)
        return np.where(self.iron, self.nu0 * (self.k1 * e + self.k3), self.nu0)

    def dnu_ds2(self, s2):
        e = np.exp(self.k2 * s2)
        return np.where(self.iron, self.nu0 * self.k1 * self.k2 * e, 0.0)

    def operator(self, u):
        """N(u)_i = sum_e area nu(|g|^2) (grad phi_i . g)."""
        gx, gy = self.gradients(u)
        nu = self.nu(gx * gx + gy * gy)
        fl = (nu * self.mesh.area)[:, None] * (self.mesh.gb * gx[:, None]
                                               + self.mesh.gc * gy[:, None])
        return self.mesh.assemble_vec(fl)

    def jacobian(self, u, inv_dt):
        gx, gy = self.gradients(u)
        s2 = gx * gx + gy * gy
        nu, dn = self.nu(s2), self.dnu_ds2(s2)
        m = self.mesh
        w = m.gb * gx[:, None] + m.gc * gy[:, None]      # G^T g per element
        Je = m.stiffness_elem(nu) + (2.0 * dn * m.area)[:, None, None] * (
            w[:, :, None] * w[:, None, :])
        return m.assemble(Je) + inv_dt * self.M

    def to_banded(self, A):
        """Upper banded storage for cholesky_banded(lower=False)."""
        u = self.bw
        n = A.shape[0]
        ab = np.zeros((u + 1, n))
        Au = sp.triu(A).tocoo()
        ab[u + Au.row - Au.col, Au.col] = Au.data
        return ab


def spec_hierarchy(spec):
    return SpatialHierarchy2D(spec["N"], spec.get("n_spatial_grids", 1),
                              spec.get("restriction", "injection"),
                              spec.get("prolongation", "bilinear"))


class FemProblem:
    """Shared plumbing, reference problems.py:70-108 in 2D."""

    n_scalars = 0

    def __init__(self, spec):
        self.spec = spec
        self.spatial = spec_hierarchy(spec)
        ex = spec.get("excitation")
        self.excitation = Excitation(**ex) if ex else None
        self.levels = [LevelModel(spec, self.spatial.cells[g])
                       for g in range(self.spatial.n_grids)]
        self._factor_cache = {}

    def initial_state(self, spatial_level=0):
        return BlockState.zeros(self.spatial.size(spatial_level), 0,
                                spatial_level)

    def loss_weights(self, spatial_level=0):
        """Lumped sigma-mass: joule_loss = sum w (du/dt)^2 ~ int sigma E^2."""
        return self.levels[spatial_level].lumped.copy()

    def source_values(self, t, smooth=False):
        lv = self.levels[0]
        if self.excitation is None:
            return np.zeros(len(lv.phases))
        f = self.excitation.smooth_value if smooth else self.excitation.value
        return np.array([float(f(ph, t)) for ph in lv.phases])

    def forcing(self, t, spatial_level=0, smooth=False):
        lv = self.levels[spatial_level]
        return self.source_values(t, smooth) @ lv.shapes


class LinearFemProblem(FemProblem):
    """Linear eddy-current step; structure of problems.py:111-146."""

    def prepare(self, spatial_level, dt):
        key = (spatial_level, float(dt))
        if key not in self._factor_cache:
            lv = self.levels[spatial_level]
            A = lv.K + lv.M * (1.0 / dt)
            self._factor_cache[key] = cholesky_banded(lv.to_banded(A))
        return self._factor_cache[key]

    def step(self, u_prev, t_prev, t_next, spatial_level=0, guess=None,
             smooth=False):
        dt = t_next - t_prev
        factor = self.prepare(spatial_level, dt)
        lv = self.levels[spatial_level]
        rhs = (self.forcing(t_next, spatial_level, smooth)
               + (1.0 / dt) * (lv.M @ u_prev.field))
        return (BlockState(cho_solve_banded((factor, False), rhs),
                           spatial_level=spatial_level),
                StepDiagnostics(iterations=1))

    def step_batch(self, U, t_prev, t_next, spatial_level=0, smooth=False):
        """Columns are independent steps; grouped by float(dt) so every
        group shares one cached factor (same arithmetic per column)."""
        U = np.asarray(U)
        out = np.empty_like(U)
        lv = self.levels[spatial_level]
        dts = np.asarray(t_next) - np.asarray(t_prev)
        MU = (lv.M @ U.T).T
        F = np.stack([self.forcing(float(t), spatial_level, smooth)
                      for t in t_next]) if len(t_next) else MU
        for dt in np.unique(dts):
            idx = np.nonzero(dts == dt)[0]
            factor = self.prepare(spatial_level, float(dt))
            rhs = F[idx] + (1.0 / float(dt)) * MU[idx]
            out[idx] = cho_solve_banded((factor, False), rhs.T).T
        return out


class NonlinearFemProblem(FemProblem):
    """Damped Newton per step, restating problems.py:201-244."""

    def __init__(self, spec):
        super().__init__(spec)
        nl = spec["nonlinear"]
        nt = nl.get("newton", {})
        self.newton_tol = nt.get("tol", 1e-11)
        self.newton_max_iters = nt.get("max_iters", 25)
        self.damping = nt.get("damping", 0.5)
        self.max_halvings = nt.get("max_halvings", 8)

    def step(self, u_prev, t_prev, t_next, spatial_level=0, guess=None,
             smooth=False):
        dt = t_next - t_prev
        inv_dt = 1.0 / dt
        lv = self.levels[spatial_level]
        rhs = (self.forcing(t_next, spatial_level, smooth)
               + inv_dt * (lv.M @ u_prev.field))
        scale = max(float(np.linalg.norm(rhs)), 1e-300)
        u = (guess.field if guess is not None else u_prev.field).copy()

        def res(v):
            return inv_dt * (lv.M @ v) + lv.operator(v) - rhs

        r = res(u)
        rnorm = float(np.linalg.norm(r))
        for it in range(self.newton_max_iters):
            if rnorm <= self.newton_tol * scale:
                return (BlockState(u, spatial_level=spatial_level),
                        StepDiagnostics(iterations=it))
            factor = cholesky_banded(lv.to_banded(lv.jacobian(u, inv_dt)))
            delta = cho_solve_banded((factor, False), -r)
            trial = u + delta
            r_trial = res(trial)
            t_norm = float(np.linalg.norm(r_trial))
            if t_norm >= rnorm:
                alpha = self.damping
                for _ in range(self.max_halvings):
                    trial = u + alpha * delta
                    r_trial = res(trial)
                    t_norm = float(np.linalg.norm(r_trial))
                    if t_norm < rnorm:
                        break
                    alpha *= 0.5
            u, r, rnorm = trial, r_trial, t_norm
        if rnorm <= self.newton_tol * scale:
            return (BlockState(u, spatial_level=spatial_level),
                    StepDiagnostics(iterations=self.newton_max_iters))
        raise NewtonConvergenceError(
            f"Newton stalled at t={t_next:.6g} on grid {spatial_level}: "
            f"|F|={rnorm:.3e} > {self.newton_tol:.1e} * {scale:.3e} "
            f"after {self.newton_max_iters} iterations",
            time=t_next, iterations=self.newton_max_iters)

    def step_batch(self, U, t_prev, t_next, spatial_level=0, smooth=False):
        out = np.empty_like(np.asarray(U))
        for b in range(len(U)):
            s, _ = self.step(BlockState(U[b], spatial_level=spatial_level),
                             float(t_prev[b]), float(t_next[b]),
                             spatial_level, None, smooth)
            out[b] = s.field
        return out


def surrogate_coupling(n_cells):
    """Torque weights c_i = sin(2 pi x_i) h^2 of the interior nodes (x-fastest
    numbering): the 2D form of reference problems.py:264-267."""
    N = int(n_cells)
    h = 1.0 / N
    x = (np.arange(1, N) * h)[None, :] * np.ones((N - 1, 1))
    return (np.sin(2.0 * math.pi * x) * (h * h)).reshape(-1)


class SurrogateFemProblem:
    """Saturating (or linear) field one-way coupled to rotor angle and speed,
    restating reference problems.py:247-287 (SurrogateMachineProblem) on the
    2D model: the field takes its step, then

        T = c . u_new,  omega' = (omega + dt T / I) / (1 + dt friction / I),
        theta' = theta + dt omega'.

    step_batch works on augmented rows [field | theta, omega]."""

    n_scalars = 2

    def __init__(self, spec):
        sg = spec["surrogate"]
        self.inertia = float(sg.get("inertia", 1.0))
        self.friction = float(sg.get("friction", 0.1))
        if self.inertia <= 0.0 or self.friction < 0.0:
            raise ValueError("need inertia > 0 and friction >= 0")
        base = dict(spec)
        base.pop("surrogate")
        self.base = (NonlinearFemProblem(base) if base.get("nonlinear")
                     else LinearFemProblem(base))
        self.spec = spec
        self.spatial = self.base.spatial
        self.levels = self.base.levels
        self.excitation = self.base.excitation
        self.couplings = [surrogate_coupling(self.spatial.cells[g])
                          for g in range(self.spatial.n_grids)]

    def initial_state(self, spatial_level=0):
        return BlockState.zeros(self.spatial.size(spatial_level), 2, spatial_level)

    def loss_weights(self, spatial_level=0):
        return self.base.loss_weights(spatial_level)

    def source_values(self, t, smooth=False):
        return self.base.source_values(t, smooth)

    def forcing(self, t, spatial_level=0, smooth=False):
        return self.base.forcing(t, spatial_level, smooth)

    def torque(self, field, spatial_level=0):
        return float(self.couplings[spatial_level] @ field)

    def _scalars(self, theta, omega, dt, torque):
        omega_new = ((omega + dt * torque / self.inertia)
                     / (1.0 + dt * self.friction / self.inertia))
        return theta + dt * omega_new, omega_new

    def step(self, u_prev, t_prev, t_next, spatial_level=0, guess=None, smooth=False):
        fp = BlockState(u_prev.field, spatial_level=spatial_level)
        fg = (BlockState(guess.field, spatial_level=spatial_level)
              if guess is not None else None)
        new, diag = self.base.step(fp, t_prev, t_next, spatial_level, fg, smooth)
        dt = t_next - t_prev
        theta, omega = u_prev.scalars
        th, om = self._scalars(theta, omega, dt, self.torque(new.field, spatial_level))
        return BlockState(new.field, [th, om], spatial_level), diag

    def step_batch(self, U, t_prev, t_next, spatial_level=0, smooth=False):
        U = np.asarray(U)
        n = self.spatial.size(spatial_level)
        F = self.base.step_batch(np.ascontiguousarray(U[:, :n]), t_prev, t_next,
                                 spatial_level, smooth)
        out = np.empty_like(U)
        out[:, :n] = F
        dt = np.asarray(t_next) - np.asarray(t_prev)
        for b in range(len(U)):
            out[b, n], out[b, n + 1] = self._scalars(U[b, n], U[b, n + 1], float(dt[b]),
                                                     self.torque(F[b], spatial_level))
        return out


def make_problem(spec):
    if spec.get("surrogate"):
        return SurrogateFemProblem(spec)
    return NonlinearFemProblem(spec) if spec.get("nonlinear") else LinearFemProblem(spec)


def sequential_solve(problem, times, spatial_level=0, smooth=False, g=None,
                     initial=None):
    """reference problems.py:319-339."""
    n = len(times)
    if initial is None:
        initial = (g[0].clone() if g is not None
                   else problem.initial_state(spatial_level))
    states = [initial]
    for i in range(1, n):
        u, _ = problem.step(states[-1], float(times[i - 1]), float(times[i]),
                            spatial_level, guess=states[-1], smooth=smooth)
        if g is not None:
            u.add_scaled(g[i], 1.0)
        states.append(u)
    return SpaceTimeVector(states, 0)


def joule_loss(u_prev, u_next, dt, weights):
    """reference problems.py:53-56."""
    du = (u_next.field - u_prev.field) / dt
    return float(weights @ (du * du))
