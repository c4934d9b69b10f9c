"""Host-side logic of the product (no GPU needed): decomposition, routing,
time hierarchy, storage accounting, spatial strategies, model assembly."""

import numpy as np
import pytest
import scipy.sparse as sp

from paper_1912_03106_b200 import (CycleSpec, Decomposition, StoppingCriterion,
                                   TimeHierarchy, assign_spatial_levels,
                                   build_uniform_grid, configs, plan_coarsening,
                                   qoi_change, storage_estimate)
from paper_1912_03106_b200.excitation import Excitation
from paper_1912_03106_b200.mesh import GridModel
from paper_1912_03106_b200.runtime import plan_moves
from paper_1912_03106_b200.time_hierarchy import cf_split


def test_decomposition_remainder_to_low_ranks():
    """runtime.py:31-105: whole intervals, remainder to the lowest ranks,
    F-tail to the last active rank, idle ranks allowed."""
    s = cf_split(2 ** 6 + 1, 4)          # 16 intervals
    d = Decomposition(s, 3)
    assert [d.n_units(w) for w in range(3)] == [6, 5, 5]
    assert d.owned_range(0) == (1, 25) and d.owned_range(2) == (45, 65)
    assert d.unit_owner(5) == 0 and d.unit_owner(6) == 1 and d.unit_owner(15) == 2
    tail = cf_split(18, 4)               # c = 0,4,8,12,16 ; F-tail 17
    d2 = Decomposition(tail, 2)
    assert d2.owned_range(1) == (9, 18)
    idle = Decomposition(cf_split(9, 4), 4)
    assert idle.active_ranks() == [0, 1] and idle.is_empty(3)
    assert idle.left_neighbor(1) == 0 and idle.right_neighbor(1) is None


def test_plan_moves_routes_runs():
    pts = np.arange(1, 9)
    src = [0, 0, 0, 0, 1, 1, 1, 1]
    dst = [0, 0, 1, 1, 1, 1, 1, 1]
    local, sends, recvs = plan_moves(pts, src, dst, 0)
    assert local == [(0, 1, 3)] and sends == [(1, 3, 5)] and recvs == []
    local, sends, recvs = plan_moves(pts, src, dst, 1)
    assert recvs == [(0, 3, 5)] and local == [(1, 5, 9)]


def test_time_hierarchy_and_plan():
    g = build_uniform_grid(0.0, 0.02, 2 ** 14)
    h = TimeHierarchy.build(g, [16, 16])
    assert [x.n_points for x in h.grids] == [16385, 1025, 65]
    assert np.array_equal(h[2].points, g.points[::256])
    assert h.splittings[2].factor == 16
    assert plan_coarsening(32, 1, 3, 4) == [32]
    assert plan_coarsening(128, 4, 3, 4) == [32]
    assert plan_coarsening(256, 8, 4, 2) == [32, 2, 2]


def test_storage_estimate_reference_values():
    """reference test_mgrit.py:232-237"""
    assert storage_estimate(2, 32, [4], 1) == 26
    assert storage_estimate(1, 32, [], 1, coarsest_factor=4) == 8
    assert storage_estimate(3, 128, [4, 4], 1) == 122


@pytest.mark.parametrize("strategy,expect", [("none", [0, 0, 0, 0, 0]),
                                             ("direct", [0, 1, 2, 2, 2]),
                                             ("delayed", [0, 0, 0, 1, 2])])
def test_spatial_strategies(strategy, expect):
    assert assign_spatial_levels(strategy, 5, 3) == expect


def test_specs_validate_like_reference():
    assert qoi_change([2.02], [2.0]) == pytest.approx(0.01)
    assert qoi_change([], []) == 0.0
    with pytest.raises(ValueError):
        CycleSpec(kind="W")
    with pytest.raises(ValueError):
        CycleSpec(gamma=-1)
    with pytest.raises(ValueError):
        StoppingCriterion(tolerance=0.0)
    with pytest.raises(ValueError):
        Excitation(modulation=1.5)


@pytest.mark.parametrize("make", [lambda: configs.config1(N=16),
                                  lambda: configs.config3(N=16, n_steps=64, levels=2)])
def test_product_assembly_matches_oracle(make):
    """mesh.py (stencil form) vs oracle/fem2d.py (element loop): two
    independent assemblies of M_sigma, K_nu, sources, Joule weights."""
    from oracle.fem2d import LevelModel
    spec = make()
    for N in (spec["N"], spec["N"] // 2):
        g, o = GridModel(spec, N), LevelModel(spec, N)
        M = sp.csr_matrix((g.m_val, g.col_idx, g.row_ptr), shape=(g.n, g.n))
        K = sp.csr_matrix((g.k_val, g.col_idx, g.row_ptr), shape=(g.n, g.n))
        Ko = o.mesh.assemble(o.mesh.stiffness_elem(np.where(o.iron, 0.0, o.nu0)))
        assert abs(M - o.M).max() <= 1e-15 * abs(o.M).max()
        assert abs(K - Ko).max() <= 1e-15 * abs(Ko).max()
        np.testing.assert_allclose(g.shapes, o.shapes, rtol=0, atol=1e-9)
        assert g.n_elem == int(o.iron.sum())
        # CSR hygiene expected by pg_add_level: sorted columns, diagonal present
        for i in range(0, g.n, max(1, g.n // 37)):
            cols = g.col_idx[g.row_ptr[i]:g.row_ptr[i + 1]]
            assert np.all(np.diff(cols) > 0) and i in cols


def test_excitation_table_matches_oracle():
    from oracle.excitation import Excitation as OExc
    kw = dict(kind="pwm", period=0.02, pulses=400, modulation=0.8, carrier="triangle")
    t = np.linspace(0.0, 0.02, 1025)
    a = Excitation(**kw).table([1, 2, 3], t)
    b = np.array([[OExc(**kw).value(ph, float(x)) for ph in (1, 2, 3)] for x in t])
    assert np.array_equal(a, b)


def test_hierarchy_rejects_levels_without_two_points():
    """time_hierarchy.py:135-140: a factor leaving < 2 points is an error."""
    g = build_uniform_grid(0.0, 1.0, 37)
    with pytest.raises(ValueError):
        TimeHierarchy.build(g, [4, 4, 4])
    with pytest.raises(ValueError):
        TimeHierarchy.build(g, [1])
    h = TimeHierarchy.build(g, [4, 4])          # 38 -> 10 -> 3 points, F-tails
    assert [x.n_points for x in h.grids] == [38, 10, 3]
    assert h.splittings[0].c_indices[-1] == 36 and h.splittings[2].factor == 2
