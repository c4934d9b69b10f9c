"""World-size-2 gloo run of the distributed MGRIT orchestration (boundary
exchange, restriction/ascent redistribution across ranks, coarsest gather /
scatter, rank-ordered norm) with a CPU test double for Phi.  The GPU path
uses the same code with NCCL; the analogue of reference
test_acceptance.py:229-267 (worker-count invariance)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1912_03106_b200 import configs


def _spec():
    return configs.config2(N=16, n_steps=1024, levels=3, grids=2, strategy="direct")


def _solve(transport):
    from cpu_double import CpuDoubleProblem
    from paper_1912_03106_b200 import (CycleSpec, MgritSolver, StoppingCriterion,
                                       TimeHierarchy, build_uniform_grid)
    spec = _spec()
    prob = CpuDoubleProblem(spec)
    grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    hier = TimeHierarchy.build(grid, spec["mgrit"]["factors"])
    solver = MgritSolver(prob, hier, CycleSpec(kind="V", gamma=1, max_iters=6,
                                               spatial_strategy="direct"),
                         StoppingCriterion(tolerance=1e-7), transport)
    run, sol = solver.solve(gather_solution=True)
    return run, sol, solver.storage_report()


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    from paper_1912_03106_b200 import DistTransport
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        run, sol, storage = _solve(DistTransport())
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
                 hist=np.array([run.initial_residual] + run.residual_norms),
                 iters=run.iterations,
                 sol=sol.numpy() if sol is not None else np.zeros(0),
                 storage=np.array([storage.total, storage.estimate]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_ranks_match_one_rank(tmp_path):
    from paper_1912_03106_b200 import NullTransport
    run1, sol1, st1 = _solve(NullTransport())
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    h1 = np.array([run1.initial_residual] + run1.residual_norms)
    for r in (r0, r1):
        assert int(r["iters"]) == run1.iterations
        np.testing.assert_allclose(r["hist"], h1, rtol=1e-10)
        tot, est = r["storage"]
        assert tot > 0 and est > 0
    np.testing.assert_allclose(r0["sol"], sol1.numpy(), rtol=0,
                               atol=1e-12 * np.abs(sol1.numpy()).max())


def test_engine_matches_oracle_engine():
    """Product engine (batched, rank-general) + oracle Phi == oracle engine."""
    from oracle import fem2d, mgrit as om, time_hierarchy as oth
    from paper_1912_03106_b200 import NullTransport
    run1, sol1, _ = _solve(NullTransport())
    spec = _spec()
    prob = fem2d.make_problem(spec)
    g = oth.build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    ro, so = om.mgrit_solve(prob, oth.TimeHierarchy.build(g, spec["mgrit"]["factors"]),
                            om.CycleSpec(kind="V", gamma=1, max_iters=6,
                                         spatial_strategy="direct"),
                            om.StoppingCriterion(tolerance=1e-7))
    assert ro.iterations == run1.iterations
    np.testing.assert_allclose([run1.initial_residual] + run1.residual_norms,
                               [ro.initial_residual] + ro.residual_norms, rtol=1e-10)
    np.testing.assert_allclose(sol1.numpy(), so, rtol=0, atol=1e-12 * np.abs(so).max())


@pytest.mark.parametrize("kind,nested", [("F", False), ("V", True)])
def test_cycle_variants_match_oracle_engine(kind, nested):
    """F-cycle (mgrit.py:617-626) and nested iterations (mgrit.py:659-675)."""
    from cpu_double import CpuDoubleProblem
    from oracle import fem2d, mgrit as om, time_hierarchy as oth
    from paper_1912_03106_b200 import (CycleSpec, MgritSolver, NullTransport,
                                       StoppingCriterion, TimeHierarchy, build_uniform_grid)
    spec = configs.config2(N=16, n_steps=512, levels=3, grids=2, strategy="delayed")
    grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    solver = MgritSolver(CpuDoubleProblem(spec), TimeHierarchy.build(grid, [16, 16]),
                         CycleSpec(kind=kind, gamma=1, max_iters=4, spatial_strategy="delayed",
                                   nested_iterations=nested),
                         StoppingCriterion(tolerance=1e-7), NullTransport())
    run, sol = solver.solve()
    g = oth.build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
    ro, so = om.mgrit_solve(fem2d.make_problem(spec), oth.TimeHierarchy.build(g, [16, 16]),
                            om.CycleSpec(kind=kind, gamma=1, max_iters=4,
                                         spatial_strategy="delayed", nested_iterations=nested),
                            om.StoppingCriterion(tolerance=1e-7))
    assert run.iterations == ro.iterations
    np.testing.assert_allclose([run.initial_residual] + run.residual_norms,
                               [ro.initial_residual] + ro.residual_norms, rtol=1e-10)
    np.testing.assert_allclose(sol.numpy(), so, rtol=0, atol=1e-12 * np.abs(so).max())


# --- worker-count invariance on a deep hierarchy (reference acceptance test 7,
# test_acceptance.py:229-267: 5 levels, p = 1, 2, 4) -------------------------------

def _spec5():
    return configs.config2(N=16, n_steps=320, levels=5, grids=2, strategy="delayed")


def _solve5(transport):
    from cpu_double import CpuDoubleProblem
    from paper_1912_03106_b200 import (CycleSpec, MgritSolver, StoppingCriterion,
                                       TimeHierarchy, build_uniform_grid)
    spec = _spec5()
    grid = build_uniform_grid(0.0, spec["tf"] * 320 / 2 ** 14, spec["n_steps"])
    # ragged on purpose: 320 = 2 * 2 * 2 * 2 * 20 leaves F-tails and ranks
    # without intervals on the coarse levels
    solver = MgritSolver(CpuDoubleProblem(spec), TimeHierarchy.build(grid, [3, 2, 2, 2]),
                         CycleSpec(kind="V", gamma=1, max_iters=8, spatial_strategy="delayed"),
                         StoppingCriterion(tolerance=1e-9), transport)
    return solver.solve(gather_solution=True)


def _worker5(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    from paper_1912_03106_b200 import DistTransport
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        run, sol = _solve5(DistTransport())
        np.savez(os.path.join(out_dir, f"w{world}_rank{rank}.npz"),
                 hist=np.array([run.initial_residual] + run.residual_norms),
                 iters=run.iterations,
                 sol=sol.numpy() if sol is not None else np.zeros(0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_five_level_solution_independent_of_worker_count(tmp_path, world):
    from paper_1912_03106_b200 import NullTransport
    run1, sol1 = _solve5(NullTransport())
    h1 = np.array([run1.initial_residual] + run1.residual_norms)
    mp.spawn(_worker5, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    scale = np.abs(sol1.numpy()).max()
    for r in range(world):
        z = np.load(tmp_path / f"w{world}_rank{r}.npz")
        assert int(z["iters"]) == run1.iterations
        np.testing.assert_allclose(z["hist"], h1, rtol=1e-10)
    z0 = np.load(tmp_path / f"w{world}_rank0.npz")
    assert np.abs(z0["sol"] - sol1.numpy()).max() <= 1e-10 * scale
