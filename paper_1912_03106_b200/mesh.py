"""Host-side model setup: structured P1 triangulation assembled in stencil
form (setup only -- nothing here runs per step).

Cell (ci, cj) of an N x N grid is cut along its '/' diagonal into
    lower = (ci, cj), (ci+1, cj), (ci+1, cj+1)
    upper = (ci, cj), (ci+1, cj+1), (ci, cj+1).
On these right isosceles triangles the P1 element matrices are closed-form,
so every interior row is a 7-point stencil (neighbours at dx, dy in
{(-1,-1), (0,-1), (-1,0), (0,0), (1,0), (0,1), (1,1)}); the stencils are
accumulated with array slicing over all cells at once and emitted as CSR
(x-fastest interior numbering, columns sorted).  The CPU oracle assembles
the same operators independently from generic per-element formulas
(oracle/fem2d.py); tests compare the two.

Material and source rules (per element, by centroid) are the ones of
configs.py / DESIGN.md 2.
"""

import numpy as np

# stencil neighbour offsets in increasing column order
OFFSETS = [(-1, -1), (0, -1), (-1, 0), (0, 0), (1, 0), (0, 1), (1, 1)]

# local vertex offsets of the two triangles of a cell
TRI_LOWER = [(0, 0), (1, 0), (1, 1)]
TRI_UPPER = [(0, 0), (1, 1), (0, 1)]

# closed-form P1 matrices on the reference right triangles (legs h):
# stiffness / nu (independent of h in 2D), mass / (sigma h^2)
K_LOWER = np.array([[0.5, -0.5, 0.0], [-0.5, 1.0, -0.5], [0.0, -0.5, 0.5]])
K_UPPER = np.array([[0.5, 0.0, -0.5], [0.0, 0.5, -0.5], [-0.5, -0.5, 1.0]])
M_REF = (np.ones((3, 3)) + np.eye(3)) / 24.0      # area/12 (1 + delta), area = h^2/2


def _centroids(N):
    """Element centroids exactly as mean-of-vertices (same rounding as the
    oracle's xy.mean): returns (lower_xy, upper_xy), each (N, N, 2) [cj, ci]."""
    h = 1.0 / N
    ci = np.arange(N)[None, :] * np.ones((N, 1))
    cj = np.arange(N)[:, None] * np.ones((1, N))

    def mean3(tri):
        xs = [((ci + dx) * h) for dx, _ in tri]
        ys = [((cj + dy) * h) for _, dy in tri]
        return np.stack([((xs[0] + xs[1]) + xs[2]) / 3.0,
                         ((ys[0] + ys[1]) + ys[2]) / 3.0], axis=-1)

    return mean3(TRI_LOWER), mean3(TRI_UPPER)


def _in_box(c, box):
    x0, y0, x1, y1 = box
    return (c[..., 0] >= x0) & (c[..., 0] < x1) & (c[..., 1] >= y0) & (c[..., 1] < y1)


class GridModel:
    """One spatial grid of the model: CSR operators, sources, weights."""

    def __init__(self, spec, N):
        self.N = N
        self.side = N - 1
        self.n = (N - 1) ** 2
        h = 1.0 / N
        cen = _centroids(N)
        cx, cy = spec.get("disc_center", (0.5, 0.5))
        sig, nu, iron, inside = [], [], [], []
        nl = spec.get("nonlinear")
        phases = sorted({s["phase"] for s in spec["sources"]})
        self.phases = phases
        for c in cen:
            r2 = (c[..., 0] - cx) ** 2 + (c[..., 1] - cy) ** 2
            s = np.where(r2 < spec["disc_radius"] ** 2, spec["sigma_disc"], 0.0)
            sig.append(s + spec["sigma_reg"])
            in_any = np.zeros(c.shape[:2], dtype=bool)
            loads = []
            for ph in phases:
                ld = np.zeros(c.shape[:2])
                for src in spec["sources"]:
                    if src["phase"] != ph:
                        continue
                    ib = _in_box(c, src["box"])
                    in_any |= ib
                    ld += np.where(ib, src["sign"] * spec["amplitude"], 0.0)
                loads.append(ld)
            inside.append(loads)
            if nl:
                r = np.sqrt(r2)
                iron.append((r >= nl["r_in"]) & (r <= nl["r_out"]) & ~in_any)
            else:
                iron.append(np.zeros(c.shape[:2], dtype=bool))
        self.iron = iron
        nu0 = spec["nu0"]
        # stencil coefficient planes over all (N+1)^2 nodes
        P = N + 1
        Mst = {o: np.zeros((P, P)) for o in OFFSETS}
        Kst = {o: np.zeros((P, P)) for o in OFFSETS}
        # preconditioner stiffness of the nonlinear model: iron at nu(|B| = 0)
        Kpre = {o: np.zeros((P, P)) for o in OFFSETS}
        nu_iron0 = nu0 * (nl["k1"] + nl["k3"]) if nl else nu0
        src_nodes = [np.zeros((P, P)) for _ in phases]
        area = 0.5 * h * h
        for t, (tri, Kref) in enumerate(((TRI_LOWER, K_LOWER), (TRI_UPPER, K_UPPER))):
            msc = sig[t] * h * h                         # (N, N) per cell
            ksc = np.where(iron[t], 0.0, nu0)            # iron handled matrix-free
            kpc = np.where(iron[t], nu_iron0, nu0)
            for a, (ax, ay) in enumerate(tri):
                rows = (slice(ay, ay + N), slice(ax, ax + N))
                for b, (bx, by) in enumerate(tri):
                    off = (bx - ax, by - ay)
                    Mst[off][rows] += msc * M_REF[a, b]
                    Kst[off][rows] += ksc * Kref[a, b]
                    Kpre[off][rows] += kpc * Kref[a, b]
                for k in range(len(phases)):
                    src_nodes[k][rows] += inside[t][k] * (area / 3.0)
        # interior rows -> CSR
        m = self.side
        ii, jj = np.meshgrid(np.arange(1, N), np.arange(1, N))   # [j-1, i-1]
        cols, mv, kv, kp, valid = [], [], [], [], []
        for (dx, dy) in OFFSETS:
            ni, nj = ii + dx, jj + dy
            ok = (ni >= 1) & (ni <= m) & (nj >= 1) & (nj <= m)
            valid.append(ok.reshape(-1))
            cols.append(((nj - 1) * m + (ni - 1)).reshape(-1))
            mv.append(Mst[(dx, dy)][1:N, 1:N].reshape(-1))
            kv.append(Kst[(dx, dy)][1:N, 1:N].reshape(-1))
            kp.append(Kpre[(dx, dy)][1:N, 1:N].reshape(-1))
        valid = np.stack(valid, 1)
        cols = np.stack(cols, 1)
        mv = np.stack(mv, 1)
        kv = np.stack(kv, 1)
        kp = np.stack(kp, 1)
        counts = valid.sum(1)
        self.row_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        self.col_idx = cols[valid].astype(np.int32)
        self.m_val = np.ascontiguousarray(mv[valid])
        self.k_val = np.ascontiguousarray(kv[valid])
        self.k_pre = np.ascontiguousarray(kp[valid]) if nl else None
        self.nnz = int(self.row_ptr[-1])
        self.shapes = np.stack([s[1:N, 1:N].reshape(-1) for s in src_nodes]) \
            if phases else np.zeros((0, self.n))
        # Joule-loss weights: lumped sigma-mass (row sums of M)
        self.weights = np.add.reduceat(self.m_val, self.row_ptr[:-1]) \
            if self.nnz else np.zeros(self.n)
        self._elements(spec, N, h)
        # surrogate-machine torque weights sin(2 pi x) h^2 (configs.with_surrogate)
        xs = np.arange(1, N) * h
        self.coupling = np.ascontiguousarray(
            np.tile(np.sin(2.0 * np.pi * xs) * (h * h), N - 1))

    def _elements(self, spec, N, h):
        """Iron elements for the matrix-free nonlinear operator."""
        self.n_elem = 0
        if not spec.get("nonlinear"):
            return
        dofs, geo = [], []
        m = self.side
        for t, tri in enumerate((TRI_LOWER, TRI_UPPER)):
            cj, ci = np.nonzero(self.iron[t])
            d = []
            for (dx, dy) in tri:
                x, y = ci + dx, cj + dy
                ok = (x >= 1) & (x <= m) & (y >= 1) & (y <= m)
                d.append(np.where(ok, (y - 1) * m + (x - 1), -1))
            dofs.append(np.stack(d, 1))
            # barycentric gradients: b = d/dx, c = d/dy (times 1/h)
            if t == 0:
                b = np.array([-1.0, 1.0, 0.0]) / h
                c = np.array([0.0, -1.0, 1.0]) / h
            else:
                b = np.array([0.0, 1.0, -1.0]) / h
                c = np.array([-1.0, 0.0, 1.0]) / h
            g = np.concatenate([b, c, [0.5 * h * h]])
            geo.append(np.tile(g, (len(ci), 1)))
        self.elem_dof = np.ascontiguousarray(np.concatenate(dofs).astype(np.int32))
        self.elem_geo = np.ascontiguousarray(np.concatenate(geo))
        self.n_elem = len(self.elem_dof)
        # node -> (element, local vertex) adjacency, CSR
        e_idx = np.repeat(np.arange(self.n_elem), 3)
        loc = np.tile(np.arange(3), self.n_elem)
        node = self.elem_dof.reshape(-1)
        ok = node >= 0
        order = np.lexsort((e_idx[ok], node[ok]))
        nodes_sorted = node[ok][order]
        self.node_elem = (e_idx[ok][order] * 4 + loc[ok][order]).astype(np.int32)
        cnt = np.bincount(nodes_sorted, minlength=self.n)
        self.node_elem_ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)


def build_grids(spec):
    """Grid models for every spatial level (N, N/2, ...)."""
    N = spec["N"]
    out = []
    for g in range(spec.get("n_spatial_grids", 1)):
        out.append(GridModel(spec, N >> g))
    return out
