"""Time grids and C/F splittings (oracle).  Follows reference
time_hierarchy.py:76-82 (linspace grid), :50-73 (C every m-th point),
:128-149 (coarse grids by slicing, coarsest reuses the last factor)."""

import numpy as np


class TimeGrid:
    def __init__(self, level, points):
        self.level = int(level)
        self.points = np.asarray(points, dtype=float)
        if self.points.ndim != 1 or self.points.size < 2:
            raise ValueError("a time grid needs at least 2 points")

    @property
    def n_points(self):
        return int(self.points.size)

    @property
    def n_steps(self):
        return int(self.points.size - 1)


class CFSplitting:
    def __init__(self, n_points, factor):
        if factor < 2:
            raise ValueError("splitting factor must be >= 2")
        self.n_points = int(n_points)
        self.factor = int(factor)
        self.c_indices = np.arange(0, n_points, factor)
        mask = np.zeros(n_points, dtype=bool)
        mask[self.c_indices] = True
        self.f_indices = np.nonzero(~mask)[0]

    @property
    def n_intervals(self):
        return int(self.c_indices.size - 1)


def build_uniform_grid(t0, tf, n_steps):
    if not tf > t0 or n_steps < 1:
        raise ValueError("bad grid")
    return TimeGrid(0, np.linspace(t0, tf, n_steps + 1))


class TimeHierarchy:
    def __init__(self, grids, factors, splittings):
        self.grids = tuple(grids)
        self.factors = tuple(factors)
        self.splittings = tuple(splittings)

    @classmethod
    def build(cls, fine_grid, factors, coarsest_factor=None):
        grids = [fine_grid]
        for m in factors:
            if m < 2:
                raise ValueError("inter-level factor must be >= 2")
            pts = grids[-1].points[::m]
            if pts.size < 2:
                raise ValueError("coarse level too small")
            grids.append(TimeGrid(len(grids), pts))
        factors = tuple(int(m) for m in factors)
        if coarsest_factor is None:
            coarsest_factor = factors[-1] if factors else 2
        lf = factors + (int(coarsest_factor),)
        spl = tuple(CFSplitting(g.n_points, lf[i]) if g.n_points > lf[i]
                    else CFSplitting(g.n_points, max(2, g.n_points - 1))
                    for i, g in enumerate(grids))
        return cls(grids, factors, spl)

    @property
    def n_levels(self):
        return len(self.grids)

    def __getitem__(self, level):
        return self.grids[level]
