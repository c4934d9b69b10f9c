"""Nested 2D grid transfers (oracle).

Tensor-product analogue of reference spatial.py:20-106.  Level g has
N_g = N / 2^g cells per side and (N_g - 1)^2 interior (Dirichlet) nodes,
numbered x-fastest: dof(i, j) = (j - 1) (N_g - 1) + (i - 1), 1 <= i, j < N_g.
Coarse node (I, J) coincides with fine node (2I, 2J) -- the 2D form of the
reference's `field[1::2]` (spatial.py:71).

restriction  : "injection"      (spatial.py:64-71, per dimension)
               "full-weighting" (BASELINE config 2; 1/16 [1 2 1; 2 4 2; 1 2 1])
prolongation : "bilinear"       (spatial.py:73-84, per dimension; config 2)
               "p1"             (nodal interpolation on the '/'-diagonal
                                 triangulation)
Scalars ride along unchanged in both directions (spatial.py:71, :84).
"""

import numpy as np

from .state import BlockState

STRATEGIES = ("none", "direct", "delayed")


class SpatialHierarchy2D:
    def __init__(self, n_cells, n_grids=1, restriction="injection",
                 prolongation="bilinear"):
        if n_grids < 1:
            raise ValueError("n_grids must be >= 1")
        cells = [int(n_cells)]
        for _ in range(n_grids - 1):
            if cells[-1] % 2 or cells[-1] < 4:
                raise ValueError(f"{cells[-1]} cells cannot be coarsened")
            cells.append(cells[-1] // 2)
        if restriction not in ("injection", "full-weighting"):
            raise ValueError(restriction)
        if prolongation not in ("bilinear", "p1"):
            raise ValueError(prolongation)
        self.cells = tuple(cells)
        self.sizes = tuple((c - 1) ** 2 for c in cells)
        self.restriction = restriction
        self.prolongation = prolongation

    @property
    def n_grids(self):
        return len(self.sizes)

    def size(self, grid):
        return self.sizes[grid]

    def side(self, grid):
        return self.cells[grid] - 1

    def spacing(self, grid):
        return 1.0 / self.cells[grid]

    def _check(self, state, grid):
        if state.spatial_level != grid or state.field.size != self.sizes[grid]:
            raise ValueError("state does not live on the expected grid")

    def _padded(self, field, grid):
        m = self.side(grid)
        p = np.zeros((m + 2, m + 2))
        p[1:-1, 1:-1] = field.reshape(m, m)
        return p

    def restrict_field(self, field, grid):
        """grid -> grid + 1."""
        p = self._padded(field, grid)          # p[j, i], 0..m+1
        mc = self.side(grid + 1)
        J = 2 * np.arange(1, mc + 1)
        if self.restriction == "injection":
            return p[np.ix_(J, J)].reshape(-1).copy()
        out = np.zeros((mc, mc))
        for dj, wj in ((-1, 1.0), (0, 2.0), (1, 1.0)):
            for di, wi in ((-1, 1.0), (0, 2.0), (1, 1.0)):
                out += (wj * wi / 16.0) * p[np.ix_(J + dj, J + di)]
        return out.reshape(-1)

    def prolong_field(self, field, grid):
        """grid -> grid - 1."""
        pc = self._padded(field, grid)         # coarse padded, 0..mc+1
        mf = self.side(grid - 1)
        # fine padded array, coarse values at even (j, i), zeros on boundary
        F = np.zeros((mf + 2, mf + 2))
        F[0::2, 0::2] = pc
        # odd i, even j: midpoint of a horizontal coarse edge
        F[0::2, 1::2] = 0.5 * (F[0::2, 0:-1:2] + F[0::2, 2::2])
        # even i, odd j: midpoint of a vertical coarse edge
        F[1::2, 0::2] = 0.5 * (F[0:-1:2, 0::2] + F[2::2, 0::2])
        # odd, odd: coarse cell centre
        ll, lr = F[0:-1:2, 0:-1:2], F[0:-1:2, 2::2]
        ul, ur = F[2::2, 0:-1:2], F[2::2, 2::2]
        if self.prolongation == "bilinear":
            F[1::2, 1::2] = 0.25 * (ll + lr + ul + ur)
        else:  # P1 on the '/' diagonal: average of its two end nodes
            F[1::2, 1::2] = 0.5 * (ll + ur)
        return F[1:-1, 1:-1].reshape(-1).copy()

    def restrict_state(self, state):
        s = state.spatial_level
        if s + 1 >= self.n_grids:
            raise ValueError("no grid below")
        self._check(state, s)
        return BlockState(self.restrict_field(state.field, s),
                          state.scalars.copy(), s + 1)

    def prolong_error(self, state):
        s = state.spatial_level
        if s == 0:
            raise ValueError("already on the finest grid")
        self._check(state, s)
        return BlockState(self.prolong_field(state.field, s),
                          state.scalars.copy(), s - 1)


def assign_spatial_levels(strategy, n_time_levels, n_spatial_grids):
    """Reference spatial.py:87-106."""
    if strategy not in STRATEGIES:
        raise ValueError(strategy)
    if strategy == "none":
        return [0] * n_time_levels
    if strategy == "direct":
        return [min(l, n_spatial_grids - 1) for l in range(n_time_levels)]
    off = max(n_time_levels - n_spatial_grids, 0)
    return [min(max(0, l - off), n_spatial_grids - 1)
            for l in range(n_time_levels)]
