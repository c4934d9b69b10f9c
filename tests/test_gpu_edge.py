"""Edge cases on the GPU path: ragged time grids (F-tails), degenerate
levels, one-level hierarchies, empty batches, aliasing / argument errors,
Newton failure bookkeeping, exact-solution fixed point -- each against the
CPU oracle engine (reference mgrit.py semantics)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _both(spec, factors, n_steps, cycle_kw, tol=1e-7, inner="cholesky", initial=None,
          t_end=None):
    from oracle import fem2d, mgrit as om, time_hierarchy as oth
    from paper_1912_03106_b200 import (CycleSpec, GpuFemProblem, StoppingCriterion,
                                       TimeHierarchy, build_uniform_grid, mgrit_solve)
    tf = t_end or spec["tf"]
    gp = GpuFemProblem(spec, inner=inner)
    grid = build_uniform_grid(0.0, tf, n_steps)
    run, sol = mgrit_solve(gp, TimeHierarchy.build(grid, factors), CycleSpec(**cycle_kw),
                           StoppingCriterion(tolerance=tol), initial_guess=initial)
    og = oth.build_uniform_grid(0.0, tf, n_steps)
    ro, so = om.mgrit_solve(fem2d.make_problem(spec), oth.TimeHierarchy.build(og, factors),
                            om.CycleSpec(**cycle_kw), om.StoppingCriterion(tolerance=tol),
                            initial_guess=None if initial is None else
                            type("T", (), {"__getitem__": lambda s, i: type(
                                "S", (), {"field": np.asarray(initial[i])})()})())
    return run, sol, ro, so


def _check(run, sol, ro, so, hist_rtol=1e-8):
    assert run.iterations == ro.iterations
    assert run.converged == ro.converged
    # Phi noise floor: two fp64 direct solves agree to ~1e-16 |u| per point
    floor = 1e-15 * np.abs(so).max() * np.sqrt(so.shape[0])
    np.testing.assert_allclose([run.initial_residual] + run.residual_norms,
                               [ro.initial_residual] + ro.residual_norms, rtol=hist_rtol,
                               atol=floor)
    s = sol.cpu().numpy()
    assert np.linalg.norm(s - so) <= 1e-9 * np.linalg.norm(so)


def _spec(N=16):
    from paper_1912_03106_b200 import configs
    return configs.config2(N=N, n_steps=64, levels=2, grids=2, strategy="direct")


@pytest.mark.parametrize("n_steps,factors", [(100, [16]), (250, [8, 4]), (37, [4, 4])])
def test_ragged_grids_with_f_tails(cuda, n_steps, factors):
    """C-points every m-th index with F-only tails (time_hierarchy.py:50-73)
    and coarsest levels whose splitting degenerates (:142-148)."""
    cyc = dict(kind="V", gamma=1, max_iters=12, spatial_strategy="direct")
    _check(*_both(_spec(), factors, n_steps, cyc, t_end=0.02 * n_steps / 1024))


def test_one_level_hierarchy_is_sequential(cuda):
    """n_levels == 1: plain sequential walk (mgrit.py:637-655)."""
    cyc = dict(kind="V", gamma=1, max_iters=3)
    run, sol, ro, so = _both(_spec(), [], 40, cyc, t_end=0.02 * 40 / 1024)
    assert run.iterations == 1 and run.converged
    _check(run, sol, ro, so)


def test_two_level_kind_ignores_deeper_levels(cuda):
    cyc = dict(kind="two-level", gamma=1, max_iters=10, spatial_strategy="none")
    _check(*_both(_spec(), [8, 4, 2], 128, cyc, t_end=0.02 * 128 / 1024))


def test_f_relaxation_only(cuda):
    cyc = dict(kind="V", gamma=0, max_iters=8, spatial_strategy="none")
    _check(*_both(_spec(), [8], 128, cyc, t_end=0.02 * 128 / 1024))


def test_exact_solution_is_a_fixed_point(cuda):
    """One cycle from the sequential solution moves it by < 1e-9
    (reference test_acceptance.py:171-191)."""
    from paper_1912_03106_b200 import (CycleSpec, GpuFemProblem, StoppingCriterion,
                                       TimeHierarchy, build_uniform_grid, mgrit_solve,
                                       sequential_solve)
    spec = _spec()
    gp = GpuFemProblem(spec, inner="cholesky")
    grid = build_uniform_grid(0.0, 0.02 * 256 / 1024, 256)
    seq = sequential_solve(gp, grid.points)
    for kind in ("V", "F"):
        run, sol = mgrit_solve(gp, TimeHierarchy.build(grid, [4, 4]),
                               CycleSpec(kind=kind, gamma=1, max_iters=1,
                                         spatial_strategy="direct"),
                               StoppingCriterion(tolerance=1e-300), initial_guess=seq)
        assert run.iterations == 1
        assert float((sol - seq).abs().max() / seq.abs().max()) < 1e-9


def test_empty_batch_and_argument_errors(cuda):
    from paper_1912_03106_b200 import GpuFemProblem
    gp = GpuFemProblem(_spec(), inner="cholesky")
    n = gp.spatial.size(0)
    dev = gp.device
    U = torch.zeros(0, n, dtype=torch.float64, device=dev)
    e = torch.zeros(0, dtype=torch.float64, device=dev)
    gp.phi_batch(0, U, e, torch.zeros(0, gp.n_src, dtype=torch.float64, device=dev), U.clone())
    U = torch.zeros(2, n, dtype=torch.float64, device=dev)
    inv = torch.full((2,), 1e4, dtype=torch.float64, device=dev)
    src = torch.zeros(2, gp.n_src, dtype=torch.float64, device=dev)
    with pytest.raises(ValueError):
        gp.phi_batch(0, U, inv, src, U)                     # aliasing
    with pytest.raises(ValueError):
        gp.phi_batch(7, U, inv, src, torch.empty_like(U))    # no such grid
    with pytest.raises(ValueError):
        gp.spatial.prolong_error(gp.initial_state(0))        # finest grid
    from paper_1912_03106_b200 import BlockState
    with pytest.raises(ValueError):
        gp.step(BlockState(torch.zeros(5, dtype=torch.float64, device=dev)), 0.0, 1e-4)


def test_newton_failure_is_recorded_not_raised(cuda):
    """Single worker: NewtonConvergenceError becomes run.failure
    (mgrit.py:706-731, reference test_mgrit.py:317-327)."""
    from paper_1912_03106_b200 import (CycleSpec, GpuFemProblem, StoppingCriterion,
                                       TimeHierarchy, build_uniform_grid, configs, mgrit_solve)
    spec = configs.config3(N=16, n_steps=64, levels=2, grids=1, strategy="none")
    spec["nonlinear"]["newton"].update(max_iters=1, tol=1e-16)
    gp = GpuFemProblem(spec)
    grid = build_uniform_grid(0.0, 0.02 * 8 / 1024, 8)
    run, sol = mgrit_solve(gp, TimeHierarchy.build(grid, [2]),
                           CycleSpec(kind="V", gamma=1, max_iters=3))
    assert not run.converged
    assert run.failure is not None and "Newton" in run.failure
    assert sol is None


def test_newton_failure_carries_time(cuda):
    """NewtonConvergenceError.time = t_next of the failing step, as the
    reference raises it (problems.py:240-244): through step() and through the
    engine's batched sweeps."""
    from paper_1912_03106_b200 import (BlockState, CycleSpec, GpuFemProblem, MgritSolver,
                                       NewtonConvergenceError, StoppingCriterion,
                                       TimeHierarchy, build_uniform_grid, configs)
    spec = configs.config3(N=16, n_steps=64, levels=2, grids=1, strategy="none")
    spec["nonlinear"]["newton"].update(max_iters=1, tol=1e-16)
    gp = GpuFemProblem(spec)
    n = gp.spatial.size(0)
    u = BlockState(torch.zeros(n, dtype=torch.float64, device=gp.device))
    with pytest.raises(NewtonConvergenceError) as ei:
        gp.step(u, 0.001, 0.0015, 0)
    assert ei.value.time == pytest.approx(0.0015)
    assert "t=0.0015" in str(ei.value)
    grid = build_uniform_grid(0.0, 0.02 * 8 / 1024, 8)
    solver = MgritSolver(gp, TimeHierarchy.build(grid, [2]), CycleSpec(kind="V", max_iters=3),
                         StoppingCriterion())
    with pytest.raises(NewtonConvergenceError) as ei:
        solver._phi_off(solver.levels[0], solver.levels[0].c_store, 1, solver.levels[0].w[0])
    assert ei.value.time is not None and ei.value.time in set(float(t) for t in grid.points)


def test_pcg_max_iters_is_an_error(cuda):
    """An unconverged Jacobi-PCG Phi is refused (PG_ENOCONV ->
    InnerSolveError), never handed to the engine as a result."""
    from paper_1912_03106_b200 import GpuFemProblem, InnerSolveError, configs
    spec = configs.config5(N=32)
    spec["inner"]["max_iters"] = 3
    prob = GpuFemProblem(spec, inner="pcg")
    n = prob.spatial.size(0)
    B = 4
    U = torch.randn(B, n, dtype=torch.float64, device=prob.device)
    out = torch.empty_like(U)
    with pytest.raises(InnerSolveError):
        prob.phi_batch(0, U, torch.full((B,), 1.0 / spec["dt"], dtype=torch.float64,
                                        device=prob.device),
                       torch.zeros(B, 0, dtype=torch.float64, device=prob.device), out)
